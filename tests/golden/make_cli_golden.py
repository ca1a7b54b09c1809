"""Golden reports of the reference CLI (burstsim/cli.py comm / balance / checkpoint / lmhead) for tests/test_cli.py.

Run in the build container (reads /root/reference, read-only):
    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_cli_golden.py
"""
import contextlib
import io
import json
from pathlib import Path

from burstsim.cli import main

CASES = {
    "comm_default": ["comm"],
    "comm_1m_2x4": ["comm", "--seq", "1048576", "--dim", "4096", "--gpus", "4", "--nodes", "2"],
    "comm_128k_8": ["comm", "--seq", "131072", "--dim", "128", "--gpus", "8", "--bw-intra-elements-per-s", "4.5e11"],
    "balance_default": ["balance"],
    "balance_zigzag_causal_16_4": ["balance", "--seq", "16", "--gpus", "4"],
    "balance_striped_window": ["balance", "--seq", "64", "--gpus", "4", "--layout", "striped", "--mask", "sliding_window",
                               "--window-tokens", "10"],
    "balance_contiguous_full": ["balance", "--seq", "32", "--gpus", "8", "--layout", "contiguous", "--mask", "full"],
    "balance_block_striped_block_sparse": ["balance", "--seq", "64", "--gpus", "2", "--layout", "block_striped",
                                           "--mask", "block_sparse", "--block-len-tokens", "8",
                                           "--block-window-tokens", "24"],
    "bad_comm_divisibility": ["comm", "--seq", "10", "--gpus", "4"],
    "checkpoint_default": ["checkpoint"],
    "checkpoint_window_64": ["checkpoint", "--seq", "64", "--dim", "8", "--mask", "sliding_window",
                             "--window-tokens", "12", "--checkpoint-split", "0.25"],
    "checkpoint_full_32": ["checkpoint", "--seq", "32", "--mask", "full", "--checkpoint-split", "0.75"],
    "bad_checkpoint_cap": ["checkpoint", "--seq", "128"],
    "lmhead_default": ["lmhead"],
    "lmhead_64_16_257": ["lmhead", "--seq", "64", "--dim", "16", "--vocab", "257", "--row-tile", "8",
                         "--vocab-tile", "32", "--seed", "3"],
    "lmhead_ragged_tiles": ["lmhead", "--seq", "13", "--dim", "5", "--vocab", "29", "--row-tile", "4",
                            "--vocab-tile", "7", "--seed", "11"],
    "bad_lmhead_sizes": ["lmhead", "--seq", "0", "--vocab-tile", "-1"],
    "verify_default": ["verify"],
}
out = {}
for name, argv in CASES.items():
    for fmt in ("json", "csv", "table"):
        so, se = io.StringIO(), io.StringIO()
        with contextlib.redirect_stdout(so), contextlib.redirect_stderr(se):
            rc = main(argv + ["--format", fmt])
        out[f"{name}/{fmt}"] = {"argv": argv + ["--format", fmt], "rc": rc, "stdout": so.getvalue(), "stderr": se.getvalue()}
Path(__file__).with_name("cli_golden.json").write_text(json.dumps(out, indent=1) + "\n")
print(f"wrote {len(out)} cases")
