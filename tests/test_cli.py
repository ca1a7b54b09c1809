"""`python -m paper_2509_19836_b200 comm|balance` reproduces the reference CLI's reports byte for
byte (json / csv / table, exit codes and error lines), against golden outputs of
burstsim/cli.py made by tests/golden/make_cli_golden.py."""

import contextlib
import io
import json
from pathlib import Path

import pytest

from paper_2509_19836_b200.cli import main

GOLDEN = json.loads((Path(__file__).parent / "golden" / "cli_golden.json").read_text())


HOST_ONLY = sorted(n for n in GOLDEN if not n.startswith(("checkpoint_", "lmhead_", "verify_")))
LMHEAD_JSON = sorted(n for n in GOLDEN if n.startswith("lmhead_") and n.endswith("/json"))
CHECKPOINT_JSON = sorted(n for n in GOLDEN if n.startswith("checkpoint_") and n.endswith("/json"))


@pytest.mark.parametrize("name", CHECKPOINT_JSON)
def test_checkpoint_plan_matches_reference(name):
    """checkpoint: params and the plan section are bit-identical (host logic); the toy run's
    gradients come from the GPU kernels, so --no-toy leaves it out on the CPU."""
    case = GOLDEN[name]
    so = io.StringIO()
    with contextlib.redirect_stdout(so):
        rc = main(case["argv"] + ["--no-toy"])
    assert rc == case["rc"] == 0
    got, want = json.loads(so.getvalue()), json.loads(case["stdout"])
    assert {k: got[k] for k in ("schema_version", "command", "seed", "params")} == \
        {k: want[k] for k in ("schema_version", "command", "seed", "params")}
    assert got["sections"][0] == want["sections"][0] and got["sections"][0]["name"] == "plan"


@pytest.mark.parametrize("name", HOST_ONLY)
def test_cli_report_matches_reference(name):
    case = GOLDEN[name]
    so, se = io.StringIO(), io.StringIO()
    with contextlib.redirect_stdout(so), contextlib.redirect_stderr(se):
        rc = main(case["argv"])
    assert rc == case["rc"]
    assert so.getvalue() == case["stdout"]
    assert se.getvalue() == case["stderr"]


def test_timeline_needs_a_gpu_or_reports_one(tmp_path):
    import torch

    if torch.cuda.is_available():
        pytest.skip("covered by the GPU suite")
    se = io.StringIO()
    with contextlib.redirect_stderr(se):
        rc = main(["timeline", "--seq", "64", "--dim", "8", "--format", "json"])
    assert rc == 2 and "needs a CUDA device" in se.getvalue()


@pytest.mark.gpu
@pytest.mark.parametrize("pass_kind", ["forward", "burst_backward"])
def test_timeline_is_measured_on_the_gpu(pass_kind):
    """The timeline subcommand runs one ring pass on the GPU(s) and reports CUDA-event times in
    the reference's schema; its traffic section equals the reference's element model."""
    from paper_2509_19836_b200.fabric import account_attention_comm

    so = io.StringIO()
    with contextlib.redirect_stdout(so):
        rc = main(["timeline", "--seq", "4096", "--dim", "128", "--gpus", "2", "--pass", pass_kind, "--format", "json"])
    assert rc == 0
    doc = json.loads(so.getvalue())
    assert doc["schema_version"] == 1 and doc["params"]["makespan_seconds"] > 0
    sec = {s["name"]: s for s in doc["sections"]}
    kinds = {row[1] for row in sec["events"]["rows"]}
    assert "compute" in kinds
    assert all(row[3] >= row[2] >= 0 for row in sec["events"]["rows"])
    for dev, intra, inter, _recv in sec["traffic"]["rows"]:  # per device, reference element model
        assert intra + inter == account_attention_comm(pass_kind, 4096, 128, 2)


@pytest.mark.gpu
def test_checkpoint_toy_run_on_the_gpu():
    """With a GPU the checkpoint report carries the toy run: every policy's gradients match the
    store-everything baseline (the reference's matches_baseline == "yes")."""
    so = io.StringIO()
    with contextlib.redirect_stdout(so):
        rc = main(["checkpoint", "--format", "json"])
    assert rc == 0
    doc = json.loads(so.getvalue())
    toy = {s["name"]: s for s in doc["sections"]}["toy_run"]
    want = json.loads(GOLDEN["checkpoint_default/json"]["stdout"])
    want_toy = {s["name"]: s for s in want["sections"]}["toy_run"]
    assert [r[0] for r in toy["rows"]] == [r[0] for r in want_toy["rows"]]
    assert [r[1] for r in toy["rows"]] == [r[1] for r in want_toy["rows"]]  # recomputed pairs: exact
    assert all(r[3] == "yes" for r in toy["rows"])


@pytest.mark.gpu
@pytest.mark.parametrize("name", LMHEAD_JSON)
def test_lmhead_report_on_the_gpu(name):
    """lmhead (cli.py:444-511): params, total loss and the footprint section as the reference
    reports them; the fused head is bf16 on the tensor cores, so its distance from the fp64 naive
    head is bf16-sized (the reference's is ~1e-16); the fp64 naive head's finite-difference check
    reproduces the reference's figure."""
    g = GOLDEN[name]
    so = io.StringIO()
    with contextlib.redirect_stdout(so):
        rc = main(g["argv"])
    assert rc == g["rc"] == 0
    doc, want = json.loads(so.getvalue()), json.loads(g["stdout"])
    assert doc["params"] == want["params"] and doc["command"] == want["command"] == "lmhead"
    sec = {s["name"]: s for s in doc["sections"]}
    ref = {s["name"]: s for s in want["sections"]}
    assert sec["footprint_elements"] == ref["footprint_elements"]
    got, exp = dict(sec["equivalence"]["rows"]), dict(ref["equivalence"]["rows"])
    assert abs(got["total_loss_nats"] - exp["total_loss_nats"]) <= 2e-3 * max(1.0, abs(exp["total_loss_nats"]))
    for key in ("max_abs_loss_diff", "max_abs_dh_diff", "max_abs_dw_diff"):
        assert got[key] < 3e-2, key
    # the fp64 naive head's finite-difference figure is the reference's own (measured: 7.5e-9 apart)
    assert abs(got["finite_difference_rel_err"] - exp["finite_difference_rel_err"]) <= 1e-4 * exp["finite_difference_rel_err"] + 1e-9


@pytest.mark.gpu
def test_verify_battery_on_the_gpu():
    """verify (cli.py:282-295): every check of the battery passes on the GPU engine (exit 0);
    the check names are the reference's, minus its simulator / cost-model checks."""
    so = io.StringIO()
    with contextlib.redirect_stdout(so):
        rc = main(["verify", "--format", "json"])
    doc = json.loads(so.getvalue())
    rows = {s["name"]: s for s in doc["sections"]}["checks"]["rows"]
    assert rc == 0, [r for r in rows if r[1] != "PASS"]
    want = json.loads(GOLDEN["verify_default/json"]["stdout"])
    ref_names = [r[0] for r in {s["name"]: s for s in want["sections"]}["checks"]["rows"]]
    names = [r[0] for r in rows]
    assert set(names) <= set(ref_names) and len(names) == len(ref_names) - 6
    assert all(r[1] == "PASS" for r in rows)
