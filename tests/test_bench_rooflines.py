"""Host-side checks of bench.py's roofline arithmetic: the work a
stage's `achieved` divides by its time must be the work of the launches timed —
counters summed over the timed steps are not multiplied by the step count again."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402

PEAKS = {"hbm_gbs": 6000.0, "bf16_tflops": 1600.0, "bf16_tflops_sustained": 1400.0}


def info(steps, **kw):
    base = {"steps": steps, "n": 1000, "d": 150, "L": 64, "W": 2, "nq": 100, "T": 10, "k": 10,
            "m": 4, "scanned_pairs": 0, "lb_pairs": 0, "lb_decided_pairs": 0,
            "rerank_path": "tensor", "rerank_filter_pairs": 0, "gt_filter_pairs": 0,
            "score_bytes": 0.0, "gt_tensor": True, "traffic": {}}
    base.update(kw)
    return base


def test_tensor_filter_rate_independent_of_step_count():
    # 1e9 pairs per step, 2 launches per step, 0.5 ms per launch: 2*1e9*150/2 flop
    # per launch / 0.5 ms = 300 TFLOP/s, whether measured over 1 or 5 steps
    for steps in (1, 5):
        for slot, key in (("gt_filter", "gt_filter_pairs"), ("rerank", "rerank_filter_pairs")):
            r = bench.roofline_for(slot, 1.0 * steps, 2 * steps, info(steps, **{key: 1e9 * steps}),
                                   PEAKS, "test")
            assert abs(r["achieved"] - 300.0) < 1e-9, (slot, steps, r["achieved"])
            assert abs(r["frac"] - 300.0 / 1400.0) < 1e-12


def test_scan_popc_count():
    # W = 2: 2 POPC per pair, minus 1 on the pairs the lower bound decides, plus 1 on
    # the pairs where it ran without deciding
    steps = 3
    i = info(steps, scanned_pairs=1e9 * steps, lb_pairs=0.4e9 * steps, lb_decided_pairs=0.3e9 * steps)
    r = bench.roofline_for("scan", 1.0 * steps, steps, i, PEAKS, "test")
    popc = (2e9 - 0.6e9 + 0.4e9)
    assert abs(r["popc_per_pair"] - popc / 1e9) < 1e-12
    assert abs(r["achieved"] - popc / 1e-3 / 1e12) < 1e-9


def test_hbm_stage_bytes():
    steps = 2
    i = info(steps)
    r = bench.roofline_for("norms", 1.0 * steps, steps, i, PEAKS, "test")
    by = 1000 * 150 * 4.0 + 1000 * 8.0
    assert abs(r["achieved"] - by / 1e-3 / 1e9) < 1e-9
