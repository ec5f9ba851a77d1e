"""The benchmark harness (paper_2303_11612_b200/harness.py) against the reference's bench.cpp
contract: CSV schema and formatting, append semantics, 14-field reads, the experiment-JSON
rules (1-based order, regimes, required keys), and -- on the GPU -- a sweep whose rows carry
the reference's fields with the RE of every decomposition."""
import json
import math

import numpy as np
import pytest


def test_csv_schema_and_round_trip(lmra, tmp_path):
    from paper_2303_11612_b200 import harness as H
    assert H.csv_header(extra=False) == "algorithm,dims,ranks,K,q,alpha,T,regime,seed,re,fit,wall_time_ms,rerun,error"
    r = H.ResultRow(algorithm="alg4", dims=[10, 9, 8], ranks=[3, 3, 2], oversampling=5, power=2, alpha=0.2,
                    t_samples=[12, 13, 14], regime="nearly-optimal", seed=7, re=0.125, fit=0.875,
                    wall_time_ms=1.5, rerun=1, error="bad, input\nhere", device_ms=1.25, gbs=3.0)
    line = H.csv_line(r, extra=False)
    assert line == "alg4,10x9x8,3x3x2,5,2,0.20000000000000001,12x13x14,nearly-optimal,7,0.125,0.875,1.5,1,bad; input;here"
    p = tmp_path / "rows.csv"
    H.write_csv(str(p), [r])
    H.write_csv(str(p), [r])  # appends; header once
    text = p.read_text().splitlines()
    assert text[0] == H.csv_header() and len(text) == 3
    back = H.read_csv(str(p))
    assert len(back) == 2 and back[0].dims == [10, 9, 8] and back[0].t_samples == [12, 13, 14]
    assert back[0].re == 0.125 and back[0].error == "bad; input;here" and back[0].gbs == 3.0


def test_experiment_config_rules(lmra):
    from paper_2303_11612_b200 import harness as H
    c = H.experiment_config_from_json(json.dumps({
        "generator": {"kind": "hilbert", "dims": [8, 8, 8]}, "algorithms": ["alg1", "sthosvd"],
        "ranks": [[2, 2, 2], [3, 3, 3]], "order": [3, 1, 2], "regime": "nearly-optimal", "power": 2,
        "reps": 2, "timed": True, "timing_reps": 3, "seed": 5}))
    assert c.base.order == [2, 0, 1] and c.base.regime == "nearly_optimal" and c.base.power == 2
    assert c.reps == 2 and c.timed and c.timing_reps == 3 and c.base.seed == 5
    for bad in ({"algorithms": [], "ranks": [[1]]}, {"algorithms": ["alg1"], "ranks": []},
                {"algorithms": ["alg1"], "ranks": [[1]], "order": [0, 1]},
                {"algorithms": ["alg1"], "ranks": [[1]], "regime": "nearly_optimal"},
                {"algorithms": ["alg1"], "ranks": [[1]], "reps": 0}):
        with pytest.raises(ValueError):
            H.experiment_config_from_json(json.dumps(bad))


@pytest.mark.gpu
def test_sweep_rows(gpu_ctx, lmra, orc):
    from paper_2303_11612_b200 import harness as H
    from paper_2303_11612_b200 import device
    cfg = H.experiment_config_from_json(json.dumps({
        "generator": {"kind": "tucker_noise", "dims": [24, 20, 16], "core_dims": [4, 4, 4], "gamma": 1e-2, "seed": 3},
        "algorithms": ["alg1", "alg4", "sthosvd", "alg3"], "ranks": [[4, 4, 4]], "reps": 2,
        "regime": "nearly-optimal", "t_samples": [100, 100, 100], "timed": True, "timing_reps": 2}))
    rows = H.run_benchmark(cfg, ctx=gpu_ctx)
    assert len(rows) == 4 * 2 * 2
    x = orc.gen_tucker_noise([24, 20, 16], [4, 4, 4], 1e-2, 3)
    for r in rows:
        if r.algorithm == "alg3":
            assert r.error.startswith("unknown algorithm") and math.isnan(r.re)
            continue
        assert r.error == "" and r.dims == [24, 20, 16] and r.wall_time_ms > 0 and r.device_ms > 0
        assert r.t_samples == ([100, 100, 100] if r.algorithm == "alg4" else [])
        want = lmra.run_algorithm(r.algorithm, lmra.DenseTensor.from_flat(x, [24, 20, 16]),
                                  lmra.AlgoConfig(rank=[4, 4, 4], seed=r.seed, regime="nearly_optimal",
                                                  t_samples=[100, 100, 100]))
        import torch
        re = device.relative_error(torch.from_numpy(x).cuda(), [24, 20, 16], want.core, want.factors)
        assert abs(r.re - re) <= 1e-12 and abs(r.fit - (1 - r.re)) == 0
    assert {r.seed for r in rows} == {0, 1}
