"""bench.py's report helpers on synthetic per-point data (CPU): the roofline
object keeps achieved / peak == frac, sums roofline times over the step, and
the side legs are compacted for the JSON line."""

import json

import pytest


def test_roofline_summary_and_compact_leg(tmp_path, monkeypatch):
    import bench
    from paper_2604_26039_b200.catalog import BASELINE_MODELS

    geom = BASELINE_MODELS[bench.MODEL]
    pts = bench.sweep_points(geom)
    assert len(pts) == 27
    per_point = [{"S": p["S"], "beta": p["beta"], "us": 100.0, "megakernel_us": 90.0} for p in pts]
    step_us = 100.0 * len(pts)
    k3_bytes = sum(bench.layer_bytes(geom, p["hist"], p["S"]) for p in pts)
    roof = bench.roofline_summary(geom, pts, per_point, step_us, k3_bytes, 90.0 * len(pts))
    assert roof["frac"] == pytest.approx(roof["achieved"] / roof["peak"])
    hbm, tf, _ = bench.load_peaks()
    want = sum(max(bench.layer_bytes(geom, p["hist"], p["S"]) / hbm / 1e3,
                   bench.layer_flops(geom, p["S"]) / tf / 1e6) for p in pts) / step_us
    assert roof["frac"] == pytest.approx(want)
    assert roof["points_hbm_bound"] + roof["points_tensor_bound"] == 27
    assert 0 < roof["bytes_only_frac"] <= roof["frac"] + 1e-12
    leg = {"workload": "w" * 300, "points": [{"S": 8, "beta": 0.5, "us": 1.0, "tflops": 2.0, "extra": 3}],
           "us_geomean": 1.0}
    c = bench.compact_leg(leg, ("S", "beta", "us"))
    assert c["points_S_beta_us"] == [[8, 0.5, 1.0]] and "points" not in c and len(c["workload"]) == 120
    assert bench.compact_leg({"error": "x"}, ("S",)) == {"error": "x"}
    json.dumps(roof)


def test_compact_line_keeps_headline_and_drops_descriptions():
    """The printed JSON line stays short: nested floats to 4 significant
    digits, long descriptions only in the per-point file, headline exact."""
    import json

    import bench

    line = {"metric": "m", "value": 164.97961361312, "ms_per_step": 1.868297576904,
            "e2e": {"value": 151.99775185443, "unit": "TFLOP/s", "how": "x" * 300},
            "roofline": {"frac": 0.61905110807983, "note": "y" * 300, "traffic_source": "z" * 200},
            "dispatch": {"method": "w" * 300, "regret_mean_pct": 1.2391145478},
            "per_point_us": [[1, 0.2, 28.7]] * 27}
    out = bench.compact_line(line)
    assert out["value"] == line["value"] and out["ms_per_step"] == line["ms_per_step"]
    assert out["e2e"]["value"] == line["e2e"]["value"] and "how" not in out["e2e"]
    assert out["roofline"] == {"frac": 0.6191}
    assert out["dispatch"] == {"regret_mean_pct": 1.239}
    assert "per_point_us" not in out
    assert len(json.dumps(out)) < 300
