// Peer fabric for the multi-GPU ring (one process per GPU): CUDA IPC arenas,
// copy-engine transfers over NVLink and stream-ordered 32-bit flags.
//
// This replaces the reference's TransferStep/MessageLog "send" of a payload to the
// next ring device (fabric.py:180-226, distributed.py:176-177, 283-286): the sender's
// copy stream pushes the bytes straight into the receiver's arena slot with a
// copy-engine memcpy (no SM work, so the attention kernels keep every SM) and then
// writes the step's epoch into a flag word in the receiver's arena; the receiver's
// compute stream blocks on that flag (cuStreamWaitValue32, GEQ) before the kernel
// that reads the slot.  All flag waits are on local memory; only writes cross NVLink.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstring>
#include <mutex>

#include "bb_host.h"

namespace bb {

namespace {

// cuStreamWriteValue32 / cuStreamWaitValue32 (the _v2 entry points cudart resolves)
using StreamValueFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);

struct StreamMemOps {
  StreamValueFn write = nullptr;
  StreamValueFn wait = nullptr;
};

const StreamMemOps& memops() {
  static StreamMemOps ops;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      ops.write = reinterpret_cast<StreamValueFn>(p);
    p = nullptr;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      ops.wait = reinterpret_cast<StreamValueFn>(p);
  });
  return ops;
}

int check_cu(CUresult r, const char* what) {
  if (r == CUDA_SUCCESS) return BB_OK;
  return set_error(BB_ERR_CUDA, "%s failed (CUresult %d)", what, static_cast<int>(r));
}

}  // namespace
}  // namespace bb

using namespace bb;

extern "C" {

int32_t bb_ipc_handle_bytes(void) { return static_cast<int32_t>(sizeof(cudaIpcMemHandle_t)); }

int bb_arena_alloc(int64_t bytes, void** ptr_out) {
  if (!ptr_out || bytes <= 0) return set_error(BB_ERR_INVALID, "bb_arena_alloc: bytes must be > 0");
  *ptr_out = nullptr;
  void* p = nullptr;
  if (int rc = check_cuda(cudaMalloc(&p, static_cast<size_t>(bytes)), "cudaMalloc(arena)")) return rc;
  // Flags start at epoch 0 (nothing ready / nothing released).  The zero fill runs on a
  // private non-blocking stream and is waited for here: on the legacy stream it would queue
  // behind the caller's in-flight ring work (which may be blocked on flags of peers) and
  // could land after a peer's first flag write into this arena.
  cudaStream_t z = nullptr;
  int rc = check_cuda(cudaStreamCreateWithFlags(&z, cudaStreamNonBlocking), "cudaStreamCreate(arena)");
  if (!rc) rc = check_cuda(cudaMemsetAsync(p, 0, static_cast<size_t>(bytes), z), "cudaMemsetAsync(arena)");
  if (!rc) rc = check_cuda(cudaStreamSynchronize(z), "cudaStreamSynchronize(arena)");
  if (z) cudaStreamDestroy(z);
  if (rc) {
    cudaFree(p);
    return rc;
  }
  *ptr_out = p;
  return BB_OK;
}

int bb_arena_free(void* ptr) { return ptr ? check_cuda(cudaFree(ptr), "cudaFree(arena)") : BB_OK; }

int bb_ipc_export(const void* ptr, void* handle_out) {
  if (!ptr || !handle_out) return set_error(BB_ERR_INVALID, "bb_ipc_export: null pointer");
  cudaIpcMemHandle_t h;
  if (int rc = check_cuda(cudaIpcGetMemHandle(&h, const_cast<void*>(ptr)), "cudaIpcGetMemHandle")) return rc;
  memcpy(handle_out, &h, sizeof(h));
  return BB_OK;
}

int bb_ipc_import(const void* handle, void** ptr_out) {
  if (!handle || !ptr_out) return set_error(BB_ERR_INVALID, "bb_ipc_import: null pointer");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  *ptr_out = nullptr;
  return check_cuda(cudaIpcOpenMemHandle(ptr_out, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
}

int bb_ipc_close(void* ptr) { return ptr ? check_cuda(cudaIpcCloseMemHandle(ptr), "cudaIpcCloseMemHandle") : BB_OK; }

int bb_copy_async(void* dst, const void* src, int64_t bytes, void* stream) {
  if (bytes < 0 || (bytes > 0 && (!dst || !src))) return set_error(BB_ERR_INVALID, "bb_copy_async: bad arguments");
  if (bytes == 0) return BB_OK;
  return check_cuda(cudaMemcpyAsync(dst, src, static_cast<size_t>(bytes), cudaMemcpyDeviceToDevice,
                                    static_cast<cudaStream_t>(stream)),
                    "cudaMemcpyAsync(peer)");
}

int bb_flag_write(void* flag, uint32_t value, void* stream) {
  if (!flag || (reinterpret_cast<uintptr_t>(flag) & 3)) return set_error(BB_ERR_INVALID, "bb_flag_write: bad flag");
  const auto& ops = memops();
  if (!ops.write) return set_error(BB_ERR_UNSUPPORTED, "cuStreamWriteValue32 unavailable");
  // default flags: a memory barrier orders every earlier write of the stream (the
  // payload copy) before the flag becomes visible to the receiver
  return check_cu(ops.write(static_cast<CUstream>(stream), reinterpret_cast<CUdeviceptr>(flag), value,
                            CU_STREAM_WRITE_VALUE_DEFAULT),
                  "cuStreamWriteValue32");
}

int bb_flag_wait(const void* flag, uint32_t value, void* stream) {
  if (!flag || (reinterpret_cast<uintptr_t>(flag) & 3)) return set_error(BB_ERR_INVALID, "bb_flag_wait: bad flag");
  const auto& ops = memops();
  if (!ops.wait) return set_error(BB_ERR_UNSUPPORTED, "cuStreamWaitValue32 unavailable");
  return check_cu(ops.wait(static_cast<CUstream>(stream), reinterpret_cast<CUdeviceptr>(flag), value,
                           CU_STREAM_WAIT_VALUE_GEQ),
                  "cuStreamWaitValue32");
}

}  // extern "C"
