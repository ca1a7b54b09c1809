"""``python -m paper_2509_19836_b200`` — burstsim-compatible reports.

Six of the reference CLI's subcommands (``burstsim/cli.py:113-131``), emitting the same
``schema_version = 1`` report (``reporting.py:17,90-105``) in table / csv / json:

* ``comm``      per-pass element accounting, the Table-1 analytic times, the burst / ring
                backward traffic ratio (``cli.py:298-330``) — host logic, bit-identical;
* ``balance``   per-device and per-step unmasked-pair tables (``cli.py:333-386``) —
                host logic, bit-identical;
* ``checkpoint`` the three checkpoint policies' storage / recompute plan (``cli.py:514-583``) —
                host logic, bit-identical — and the toy run, executed on the GPU;
* ``verify``    the property battery (``cli.py:282-295``, ``verification.py``) against the
                GPU engine (``verification.py`` here: host checks exact, device checks at
                the build tolerances);
* ``lmhead``    fused vs naive LM head (``cli.py:444-511``): the fused head runs on the
                tcgen05 kernels (bf16 operands, fp32 accumulation), the naive head and the
                finite-difference check in float64 on the device (``numerics``); the
                footprint section is host logic, identical to the reference's;
* ``timeline``  the event timeline of one ring pass (``cli.py:389-441``) — MEASURED here:
                the pass runs on the local GPUs through ``run_with_schedule`` (CUDA events
                per ring step and per peer copy), where the reference simulates it.

Flag names and defaults follow the reference (``--seq``, ``--dim``, ``--gpus``, ``--nodes``,
``--layout``, ``--mask``, ``--window-tokens``, ``--block-len-tokens``,
``--block-window-tokens``, ``--schedule``, ``--format``, ``--output``, ``--seed``); bad
configurations exit 2 with one ``error: ...`` line per problem, as ``ConfigError`` does.
"""

from __future__ import annotations

import argparse
import io
import json
import sys
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

from .fabric import (
    BURST_BACKWARD,
    FORWARD,
    RING_BACKWARD,
    SCHEDULE_KINDS,
    STRATEGIES,
    OverlapSchedule,
    Topology,
    account_attention_comm,
    analytic_comm_time,
)
from .masks import MASK_KINDS, causal_mask, full_mask, sliding_window_mask, validate_mask
from .partitioning import LAYOUT_KINDS, ShardLayout, balance_report, block_mask_from_window

SCHEMA_VERSION = 1
EXIT_OK, EXIT_SUITE_FAILED, EXIT_BAD_CONFIG = 0, 1, 2


class BadConfig(Exception):
    def __init__(self, problems: list[str]):
        super().__init__("; ".join(problems))
        self.problems = problems


# ------------------------------------------------------------------------------ reports
def _plain(x):
    """numpy scalars -> Python scalars, so json / repr print the same digits as floats do."""
    if isinstance(x, (np.integer, np.bool_)):
        return int(x)
    if isinstance(x, np.floating):
        return float(x)
    return x


def _text(x) -> str:
    return repr(x) if isinstance(x, float) else str(x)


@dataclass
class Report:
    command: str
    seed: int
    params: dict
    sections: list[tuple[str, list[str], list[list]]] = field(default_factory=list)

    def section(self, name: str, headers: list[str], rows) -> None:
        self.sections.append((name, list(headers), [[_plain(v) for v in r] for r in rows]))

    def render(self, fmt: str) -> str:
        params = {k: _plain(v) for k, v in self.params.items()}
        if fmt == "json":
            doc = {"schema_version": SCHEMA_VERSION, "command": self.command, "seed": self.seed, "params": params,
                   "sections": [{"name": n, "headers": h, "rows": r} for n, h, r in self.sections]}
            return json.dumps(doc, indent=2) + "\n"
        buf = io.StringIO()
        if fmt == "csv":
            buf.write(f"# command: {self.command}\n# seed: {self.seed}\n")
            buf.writelines(f"# param {k}: {_text(v)}\n" for k, v in params.items())
            for name, headers, rows in self.sections:
                buf.write(f"# section: {name}\n" + ",".join(headers) + "\n")
                buf.writelines(",".join(_text(v) for v in r) + "\n" for r in rows)
            return buf.getvalue()
        if fmt != "table":
            raise ValueError(f"unknown output format {fmt!r}, expected table/csv/json")
        buf.write(f"# {self.command} (seed={self.seed})\n")
        buf.writelines(f"# {k} = {_text(v)}\n" for k, v in params.items())
        for name, headers, rows in self.sections:
            grid = [headers] + [[_text(v) for v in r] for r in rows]
            width = [max(len(line[c]) for line in grid) for c in range(len(headers))]
            buf.write(f"\n== {name} ==\n")
            for i, line in enumerate(grid):
                buf.write("  ".join(cell.ljust(w) for cell, w in zip(line, width)).rstrip() + "\n")
                if i == 0:
                    buf.write("  ".join("-" * w for w in width) + "\n")
        return buf.getvalue()


# ------------------------------------------------------------------------------ arguments
def _topology(a, problems) -> Topology | None:
    try:
        return Topology(num_nodes=a.nodes, gpus_per_node=a.gpus, lat_intra=a.lat_intra, lat_inter=a.lat_inter,
                        bw_intra=a.bw_intra, bw_inter=a.bw_inter)
    except ValueError as exc:
        problems.append(f"topology: {exc}")
        return None


def _mask(a, seq: int, problems):
    try:
        if a.mask == "full":
            return full_mask()
        if a.mask == "causal":
            return causal_mask()
        if a.mask == "sliding_window":
            m = sliding_window_mask(a.window if a.window is not None else max(1, seq // 2))
        else:
            bl = a.block_len if a.block_len is not None else max(1, seq // 4)
            bw = a.block_window if a.block_window is not None else 2 * bl
            m = block_mask_from_window(seq, bl, bw)
        validate_mask(m, seq)
        return m
    except ValueError as exc:
        problems.append(f"mask: {exc}")
        return None


def cmd_comm(a) -> Report:
    problems: list[str] = []
    topo = _topology(a, problems)
    g = topo.total_devices if topo else 0
    if topo and a.seq % g:
        problems.append(f"seq: device count {g} must divide sequence length {a.seq}")
    if problems:
        raise BadConfig(problems)
    rep = Report("comm", a.seed, {"seq_len_tokens": a.seq, "dim": a.dim, "devices": g, "nodes": a.nodes})
    rows = []
    for kind in (FORWARD, RING_BACKWARD, BURST_BACKWARD):
        total = account_attention_comm(kind, a.seq, a.dim, g)
        rows.append([kind, total, total // g])
    rep.section("elements_per_device", ["pass", "total_elements", "per_step_elements"], rows)
    payload = (a.seq // g) * a.dim
    rep.section("analytic_seconds", ["strategy", "seconds"], [[s, analytic_comm_time(s, topo, payload)] for s in STRATEGIES])
    rep.section("ratios", ["name", "value"], [["burst_vs_ring_backward_elements", (3 * a.dim + 2) / (4 * a.dim)]])
    return rep


def cmd_balance(a) -> Report:
    problems: list[str] = []
    mask = _mask(a, a.seq, problems)
    layout = None
    try:
        bl = None
        if a.layout == "block_striped":
            bl = a.block_len if a.block_len is not None else max(a.gpus, a.seq // 4)
        layout = ShardLayout(a.layout, a.seq, a.gpus, block_len=bl)
    except ValueError as exc:
        problems.append(f"layout: {exc}")
    if problems or mask is None or layout is None:
        raise BadConfig(problems)
    wr = balance_report(layout, mask)
    rep = Report("balance", a.seed, {"seq_len_tokens": a.seq, "devices": a.gpus, "layout": a.layout,
                                     "mask": mask.describe()})
    rep.section("per_device_totals", ["device", "unmasked_pairs"], [[i + 1, c] for i, c in enumerate(wr.per_device_pairs)])
    steps = len(wr.per_step_pairs[0])
    rep.section("per_step_pairs", ["device"] + [f"step_{t + 1}" for t in range(steps)],
                [[i + 1, *row] for i, row in enumerate(wr.per_step_pairs)])
    rep.section("spread", ["total_pairs", "device_spread", "max_step_spread"],
                [[wr.total_pairs, wr.device_spread, wr.max_step_spread]])
    return rep


def cmd_checkpoint(a) -> Report:
    from .checkpointing import FULL_RECOMPUTE, SELECTIVE_PP, SEQUENCE_SELECTIVE, CheckpointPolicy, execute_toy
    from .checkpointing import plan as checkpoint_plan

    problems: list[str] = []
    mask = _mask(a, a.seq, problems)
    if a.seq > 64:
        problems.append(f"seq: toy checkpoint runs are capped at 64 tokens, got {a.seq}")
    if problems or mask is None:
        raise BadConfig(problems)
    rep = Report("checkpoint", a.seed, {"seq_len_tokens": a.seq, "dim": a.dim, "mask": mask.describe(),
                                        "checkpoint_split": a.split})
    rows, toy_rows = [], []
    try:
        for pol in (CheckpointPolicy(FULL_RECOMPUTE), CheckpointPolicy(SELECTIVE_PP),
                    CheckpointPolicy(SEQUENCE_SELECTIVE, a.split)):
            pr = checkpoint_plan(pol, a.seq, a.dim, mask)
            rows.append([pol.kind, pr.stored_elements_per_layer, pr.attention_extra_elements, pr.recompute_pairs,
                         pr.recompute_fraction])
            if not a.no_toy:
                import torch

                if not torch.cuda.is_available():
                    raise BadConfig(["checkpoint: the toy run executes on a CUDA device (use --no-toy for the plan)"])
                toy = execute_toy(pol, a.seq, a.dim, mask, a.seed)
                toy_rows.append([pol.kind, toy.recomputed_pairs, toy.max_grad_diff,
                                 "yes" if toy.matches_baseline else "no"])
    except ValueError as exc:
        raise BadConfig([str(exc)]) from exc
    rep.section("plan", ["policy", "stored_elements_per_layer", "attention_extra_elements", "recompute_pairs",
                         "recompute_fraction"], rows)
    if not a.no_toy:
        rep.section("toy_run", ["policy", "recomputed_pairs", "max_grad_diff", "matches_baseline"], toy_rows)
    return rep


def cmd_verify(a) -> Report:
    """The property battery (reference: cli.py:282-295) on the B200 engine (``verification``)."""
    import torch

    from .verification import run_all

    if not torch.cuda.is_available():
        raise BadConfig(["verify: the property suite executes on a CUDA device (no CPU fallback)"])
    checks = run_all(a.seed)
    failed = sum(not c.passed for c in checks)
    rep = Report("verify", a.seed, {})
    rep.section("checks", ["check", "status", "detail"], [[c.name, "PASS" if c.passed else "FAIL", c.detail]
                                                           for c in checks])
    rep.section("summary", ["total", "passed", "failed"], [[len(checks), len(checks) - failed, failed]])
    rep.exit_code = EXIT_SUITE_FAILED if failed else EXIT_OK
    return rep


def cmd_lmhead(a) -> Report:
    """Fused vs naive LM head (reference: cli.py:444-511, same inputs and report sections)."""
    from .layer import finite_diff_check, naive_lmhead_loss
    from .lmhead import FusionConfig, fused_lmhead_loss, memory_footprint
    from .numerics import seeded_random_matrix

    if a.row_tile is None:
        a.row_tile = max(1, a.seq // 2 if a.seq else 4)
    if a.vocab_tile is None:
        a.vocab_tile = max(1, (a.vocab or 17) // 3)
    problems = [f"{name}: must be >= 1, got {getattr(a, name)}"
                for name in ("seq", "dim", "vocab", "row_tile", "vocab_tile") if getattr(a, name) < 1]
    if problems:
        raise BadConfig(problems)
    import torch

    if not torch.cuda.is_available():
        raise BadConfig(["lmhead: the fused and naive heads execute on a CUDA device (no CPU fallback)"])
    h = seeded_random_matrix(a.seq, a.dim, a.seed)
    w = seeded_random_matrix(a.vocab, a.dim, a.seed + 1)
    y = np.random.default_rng(a.seed + 2).integers(0, a.vocab, size=a.seq)
    cfg = FusionConfig(a.row_tile, a.vocab_tile)
    naive = naive_lmhead_loss(h, w, y)
    fused = fused_lmhead_loss(h, w, y, cfg)
    naive_elems, fused_elems = memory_footprint(a.seq, a.vocab, a.dim, cfg)
    fd_err = finite_diff_check(lambda x: float(np.sum(naive_lmhead_loss(x, w, y).loss)), h, naive.dh, h=1e-6)
    rep = Report("lmhead", a.seed, {"seq_len_tokens": a.seq, "dim": a.dim, "vocab": a.vocab,
                                    "row_tile": a.row_tile, "vocab_tile": a.vocab_tile})
    rep.section("equivalence", ["metric", "value"], [
        ["max_abs_loss_diff", float(np.max(np.abs(fused.loss - naive.loss)))],
        ["max_abs_dh_diff", float(np.max(np.abs(fused.dh - naive.dh)))],
        ["max_abs_dw_diff", float(np.max(np.abs(fused.dw - naive.dw)))],
        ["finite_difference_rel_err", fd_err],
        ["total_loss_nats", float(np.sum(fused.loss))],
    ])
    rep.section("footprint_elements", ["naive_logits", "fused_peak_model", "fused_peak_instrumented"],
                [[naive_elems, fused_elems, fused.peak_aux_elements]])
    return rep


def cmd_timeline(a) -> Report:
    """One ring pass measured on the local GPUs (reference: simulated, cli.py:389-441)."""
    problems: list[str] = []
    topo = _topology(a, problems)
    if a.seq is None:
        a.seq = 4096 * (topo.total_devices if topo else 1)
    if topo and a.seq % topo.total_devices:
        problems.append(f"seq: device count {topo.total_devices} must divide sequence length {a.seq}")
    if problems:
        raise BadConfig(problems)
    import torch

    from .distributed import run_with_schedule

    if not torch.cuda.is_available():
        raise BadConfig(["timeline: the measured timeline needs a CUDA device (no CPU fallback)"])
    g = topo.total_devices
    layout = ShardLayout(a.layout, a.seq, g)
    rng = np.random.default_rng(a.seed)
    q, k, v, do = (rng.uniform(-1, 1, (a.seq, a.dim)) for _ in range(4))
    devices = [torch.device("cuda", i % torch.cuda.device_count()) for i in range(g)]
    run = run_with_schedule(a.pass_kind, layout, causal_mask(), q, k, v, do=do if a.pass_kind != FORWARD else None,
                            topology=topo, schedule=OverlapSchedule(a.schedule), devices=devices)
    tl, log = run.timeline, run.message_log
    rep = Report("timeline", a.seed, {"schedule": a.schedule, "pass": a.pass_kind, "seq_len_tokens": a.seq,
                                      "dim": a.dim, "devices": g, "nodes": topo.num_nodes,
                                      "makespan_seconds": tl.makespan, "source": "measured (CUDA events)"})
    rep.section("events", ["device", "kind", "start_seconds", "end_seconds", "label"],
                [[e.device, e.kind, e.start, e.end, e.label] for e in tl.events])
    rep.section("traffic", ["device", "sent_intra_elements", "sent_inter_elements", "received_elements"],
                [[i, log.sent(i, "intra"), log.sent(i, "inter"), log.received(i)] for i in range(1, g + 1)])
    return rep


# ------------------------------------------------------------------------------ parser
def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="python -m paper_2509_19836_b200",
                                 description="burstsim-compatible reports backed by the B200 engine")
    sub = ap.add_subparsers(dest="command", required=True)

    def common(p):
        p.add_argument("--seed", type=int, default=0)
        p.add_argument("--format", choices=("table", "csv", "json"), default="table", dest="fmt")
        p.add_argument("--output", default=None)

    def topology(p):
        p.add_argument("--gpus", type=int, default=2)
        p.add_argument("--nodes", type=int, default=1)
        p.add_argument("--lat-intra-seconds", type=float, default=1e-6, dest="lat_intra")
        p.add_argument("--lat-inter-seconds", type=float, default=5e-6, dest="lat_inter")
        p.add_argument("--bw-intra-elements-per-s", type=float, default=1e9, dest="bw_intra")
        p.add_argument("--bw-inter-elements-per-s", type=float, default=1e8, dest="bw_inter")

    p = sub.add_parser("verify", help="run the property suite on the GPU engine")
    common(p)
    p.set_defaults(run=cmd_verify)

    p = sub.add_parser("comm", help="traffic accounting and analytic times")
    common(p)
    p.add_argument("--seq", type=int, default=8)
    p.add_argument("--dim", type=int, default=4)
    topology(p)
    p.set_defaults(run=cmd_comm)

    p = sub.add_parser("balance", help="workload balance tables")
    common(p)
    p.add_argument("--seq", type=int, default=8)
    p.add_argument("--gpus", type=int, default=2)
    p.add_argument("--layout", choices=LAYOUT_KINDS, default="zigzag")
    p.add_argument("--mask", choices=MASK_KINDS, default="causal")
    p.add_argument("--window-tokens", type=int, default=None, dest="window")
    p.add_argument("--block-len-tokens", type=int, default=None, dest="block_len")
    p.add_argument("--block-window-tokens", type=int, default=None, dest="block_window")
    p.set_defaults(run=cmd_balance)

    p = sub.add_parser("checkpoint", help="checkpoint policy plans and toy run")
    common(p)
    p.add_argument("--seq", type=int, default=16)
    p.add_argument("--dim", type=int, default=4)
    p.add_argument("--checkpoint-split", type=float, default=0.5, dest="split")
    p.add_argument("--mask", choices=MASK_KINDS, default="causal")
    p.add_argument("--window-tokens", type=int, default=None, dest="window")
    p.add_argument("--block-len-tokens", type=int, default=None, dest="block_len")
    p.add_argument("--block-window-tokens", type=int, default=None, dest="block_window")
    p.add_argument("--no-toy", action="store_true", help="plan only (the toy run needs a GPU)")
    p.set_defaults(run=cmd_checkpoint)

    p = sub.add_parser("lmhead", help="fused vs naive LM-head loss (GPU)")
    common(p)
    p.add_argument("--seq", type=int, default=8)
    p.add_argument("--dim", type=int, default=4)
    p.add_argument("--vocab", type=int, default=17)
    p.add_argument("--row-tile", type=int, default=None, dest="row_tile")
    p.add_argument("--vocab-tile", type=int, default=None, dest="vocab_tile")
    p.set_defaults(run=cmd_lmhead)

    p = sub.add_parser("timeline", help="measured event timeline of one ring pass (GPU)")
    common(p)
    p.add_argument("--schedule", choices=SCHEDULE_KINDS, default="activation")
    p.add_argument("--pass", choices=(FORWARD, RING_BACKWARD, BURST_BACKWARD), default=FORWARD, dest="pass_kind")
    p.add_argument("--seq", type=int, default=None)
    p.add_argument("--dim", type=int, default=128)
    p.add_argument("--layout", choices=LAYOUT_KINDS[:3], default="zigzag")
    topology(p)
    p.set_defaults(run=cmd_timeline)
    return ap


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    try:
        rep = args.run(args)
    except BadConfig as exc:
        for line in exc.problems:
            sys.stderr.write(f"error: {line}\n")
        return EXIT_BAD_CONFIG
    text = rep.render(args.fmt)
    if args.output:
        Path(args.output).write_text(text)
    else:
        sys.stdout.write(text)
    return getattr(rep, "exit_code", EXIT_OK)
