"""Row f4, host side (no GPU): ExperimentSpec validation and JSON form, the
CSV writer's fixed columns (experiment.py:63-133, 266-290), and the host
synthetic-input construction (synth.py:59-88) against the CPU oracle."""

import json
import os

import numpy as np
import pytest

import rsvd_oracle as o
from conftest import GOLDEN
from paper_1504_05477_b200 import ExperimentSpec, SyntheticSpec, Variant, rows_to_csv
from paper_1504_05477_b200.synth import cgs2, synth_matrix

SYN = {"n": 30, "d": 20, "spectrum": [1.0, 0.5, 0.25], "seed": 1}


def test_spec_validation():
    ok = ExperimentSpec.from_dict({"algorithms": ["BK", "si"], "k": 3, "q_list": [1, 2], "seeds": [0],
                                   "synthetic": SYN})
    assert ok.algorithms == (Variant.BLOCK_KRYLOV, Variant.SIMULTANEOUS_ITERATION)
    assert ExperimentSpec.from_dict(ok.to_dict()).to_dict() == ok.to_dict()
    bad = [dict(algorithms=[], k=3, q_list=[1], seeds=[0]),
           dict(algorithms=["bk"], k=3, q_list=[1], seeds=[]),
           dict(algorithms=["bk"], k=3, seeds=[0]),
           dict(algorithms=["bk"], k=3, q_list=[1], eps_list=[0.1], seeds=[0]),
           dict(algorithms=["bk"], k=3, q_list=[1], seeds=[0], oracle_policy="never")]
    for b in bad:
        with pytest.raises(ValueError):
            ExperimentSpec(synthetic=SyntheticSpec.from_dict(SYN), **b)
    with pytest.raises(ValueError):  # both inputs
        ExperimentSpec(algorithms=["bk"], k=3, q_list=[1], seeds=[0], input_path="x.mtx",
                       synthetic=SyntheticSpec.from_dict(SYN))
    with pytest.raises(ValueError):
        SyntheticSpec(n=5, d=5, spectrum=[1.0, 2.0])  # ascending


def test_rows_to_csv_columns():
    golden = json.load(open(os.path.join(GOLDEN, "sweep_golden.json")))
    rows = [dict(r, wall_ms=1.5) for r in golden["rows"][:2]]
    text = rows_to_csv(rows)
    lines = text.strip().split("\n")
    assert lines[0] == golden["csv_header"]
    f = lines[1].split(",")
    assert f[:5] == ["bk", "5", "5", "1", "0"] and float(f[5]) == rows[0]["frob_ratio"]


def test_host_synthetic_matches_oracle_restatement():
    spec = SyntheticSpec(n=40, d=25, spectrum=1.0 / np.arange(1, 11), seed=3)
    A = synth_matrix(spec, check=False).data
    ref = o.synth_matrix(40, 25, spec.spectrum, seed=3, mm=o.mm_blas)
    assert np.max(np.abs(A - ref)) < 1e-14
    q = cgs2(np.random.default_rng(0).standard_normal((50, 8)))
    assert np.max(np.abs(q.T @ q - np.eye(8))) < 1e-14
