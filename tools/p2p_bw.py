"""NVLink copy-engine bandwidth between two GPUs (the ring transport's link roofline):
one-directional and bidirectional D2D peer copies, 1 / 2 / 4 concurrent streams, 1 GiB."""
import json
import torch

n = 1 << 30
a0 = torch.empty(n, dtype=torch.uint8, device="cuda:0")
b1 = torch.empty(n, dtype=torch.uint8, device="cuda:1")
a1 = torch.empty(n, dtype=torch.uint8, device="cuda:1")
b0 = torch.empty(n, dtype=torch.uint8, device="cuda:0")
out = {}
for bidir in (False, True):
    for k in (1, 2, 4):
        s0 = [torch.cuda.Stream(device="cuda:0") for _ in range(k)]
        s1 = [torch.cuda.Stream(device="cuda:1") for _ in range(k)]
        part = n // k
        best = 0.0
        for _ in range(5):
            torch.cuda.synchronize("cuda:0"); torch.cuda.synchronize("cuda:1")
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record(torch.cuda.current_stream("cuda:0"))
            for i in range(k):
                s0[i].wait_event(e0)
                with torch.cuda.stream(s0[i]):
                    b1[i * part:(i + 1) * part].copy_(a0[i * part:(i + 1) * part], non_blocking=True)
                if bidir:
                    with torch.cuda.stream(s1[i]):
                        b0[i * part:(i + 1) * part].copy_(a1[i * part:(i + 1) * part], non_blocking=True)
            for i in range(k):
                torch.cuda.current_stream("cuda:0").wait_stream(s0[i])
            if bidir:
                for i in range(k):
                    s1[i].synchronize()
            e1.record(torch.cuda.current_stream("cuda:0"))
            e1.synchronize()
            t = e0.elapsed_time(e1) / 1e3
            best = max(best, (2 if bidir else 1) * n / t / 1e9)
        out[f"{'bidir' if bidir else 'unidir'}_{k}streams_GBps"] = best
print(json.dumps({"p2p_copy_engine_bandwidth": out, "bytes_per_copy": n, "peak_per_direction_GBps": 900}))
