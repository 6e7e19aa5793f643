"""CPU checks of bench.py's contract pieces that need no GPU: every workload's config and
arithmetic label, and the reference arm's JSON line on small synthetic workloads (the oracle
port of blockstat's algorithm, timed on the host)."""

import argparse
import json
import sys
from pathlib import Path

import numpy as np
import pytest

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402


@pytest.mark.parametrize("name", sorted(bench.WORKLOADS))
@pytest.mark.parametrize("n_gpus", [1, 2, 8])
def test_every_workload_has_a_config(name, n_gpus):
    wl = dict(bench.WORKLOADS[name], key=name)
    cfg = bench._config(wl, n_gpus, 20)
    assert cfg["workload"] == wl["desc"] and cfg["iterations_timed"] == 20
    assert f"over {n_gpus} GPU(s)" in cfg["partition"]
    per_gpu = bench._per_gpu_bytes(wl, n_gpus)
    if bench._flushes(wl, n_gpus):  # small per-GPU inputs: the L2 is flushed between timed iterations
        assert per_gpu < 1.5 * bench.L2_BYTES and "buffer is written between timed iterations" in cfg["l2_flush"]
    else:
        assert per_gpu >= 1.5 * bench.L2_BYTES and "exceed the 126 MB L2" in cfg["l2_flush"]
    assert bench._arith_dtype(wl) in {"f32", "f64", "int8->f32", "u2->f32", "u2->f64"}


def test_l2_policy_at_scale():
    """C1 (0.8 GB float64) streams from HBM up to 4 GPUs (0.2 GB each) and is flushed per
    iteration on 8 (0.1 GB < the L2); the headline C2 never needs a flush."""
    c1, c2 = bench.WORKLOADS["nmf_mu_c1"], bench.WORKLOADS["nmf_apg_c2"]
    assert not any(bench._flushes(c1, n) for n in (1, 2, 4)) and bench._flushes(c1, 8)
    assert not any(bench._flushes(c2, n) for n in (1, 2, 4, 8))


def test_arithmetic_labels():
    assert bench._arith_dtype(bench.WORKLOADS["cox_c5"]) == "u2->f32"
    assert bench._arith_dtype(bench.WORKLOADS["cox_c5_f64"]) == "u2->f64"
    assert bench._arith_dtype(bench.WORKLOADS["nmf_apg_c2"]) == "f32"
    assert bench._arith_dtype(bench.WORKLOADS["nmf_mu_c1"]) == "f64"


@pytest.mark.parametrize("wl", [
    dict(kind="nmf", algo="apg", m=3000, n=2500, r=6, dtype="float32", desc="tiny NMF-APG"),
    dict(kind="nmf", algo="mu", m=2000, n=800, r=4, dtype="float64", desc="tiny NMF-MU"),
    dict(kind="cox", m=3000, n=400, dtype="int8", lam=1e-8, desc="tiny Cox genotypes"),
    dict(kind="cox", m=2000, n=300, dtype="float32", lam=1e-8, desc="tiny Cox"),
])
def test_reference_arm_line(wl, capsys):
    args = argparse.Namespace(gpus=1, steps=2, warmup=1)
    bench._run_reference(args, wl)
    line = json.loads(capsys.readouterr().out.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["metric"] == "iterations/sec" and line["unit"] == "it/s"
    assert line["value"] > 0 and np.isfinite(line["value"])
    assert line["config"] == bench._config(wl, 1, 2)
    assert line["e2e"] == {"value": line["value"], "unit": "it/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    cb = line["cpu_baseline"]
    assert cb["kind"] == "port" and cb["cores"] >= 1 and cb["value"] == line["value"]
    frac = line["sample_fraction_of_iteration"]
    assert 0 < frac <= 1 and line["extrapolated"] == (frac < 1)
    # value = fraction of an iteration per measured sample second
    assert line["value"] == pytest.approx(frac / (line["ms_per_step"] / 1e3), rel=1e-9)
