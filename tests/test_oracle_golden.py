"""Pin the CPU oracle (oracle/ramp_ref.py) to the reference's own outputs.

Every fixture under tests/golden/ was produced by the reference package
itself (tests/golden/gen_golden.py); these tests run on CPU only.
"""

from __future__ import annotations

import hashlib
import json

import numpy as np
import pytest

from oracle import ramp_ref as R
from tests._util import GEOMS, golden

BASELINE_GEOMS = {
    "OLMoE-1B-7B": dict(E=64, N=2048, K=2048, top_k=8),
    "Qwen3-30B-A3B": dict(E=128, N=1536, K=2048, top_k=8),
    "Mixtral-8x7B": dict(E=8, N=28672, K=4096, top_k=2),
    "DeepSeek-V3": dict(E=256, N=4096, K=7168, top_k=8),
}
CATALOG = {
    "OLMoE": (64, 2048, 2048), "Qwen3": (128, 1536, 2048), "DSv3-EP8": (32, 512, 7168),
    "Mixtral": (8, 32768, 6144), "DSv3-TP8": (256, 512, 7168), "DBRX": (16, 21504, 6144),
}


def _geom_ENK(name):
    if name in GEOMS:
        g = GEOMS[name]
        return g["E"], g["N"], g["K"]
    if name in BASELINE_GEOMS:
        g = BASELINE_GEOMS[name]
        return g["E"], g["N"], g["K"]
    return CATALOG[name]


def test_derive_seed():
    for row in golden("seeds.json"):
        assert R.derive_seed(*row["keys"]) == int(row["seed"])


def test_sample_histogram_matches_reference():
    n = 0
    for s in golden("histograms.json")["samples"]:
        if "unreachable" in s:
            with pytest.raises(R.Unreachable):
                R.sample_histogram(s["E"], s["S"], s["top_k"], s["beta"], int(s["seed"]))
            continue
        counts, beta = R.sample_histogram(s["E"], s["S"], s["top_k"], s["beta"], int(s["seed"]))
        assert counts == s["counts"], (s["model"], s["S"], s["beta"])
        assert beta == pytest.approx(s["beta_achieved"], rel=1e-12, abs=1e-12)
        n += 1
    assert n > 300


def test_balancedness():
    for row in golden("histograms.json")["balancedness"]:
        assert R.balancedness(row["counts"]) == pytest.approx(row["beta"], rel=1e-12, abs=1e-15)


def _digest(cols):
    return hashlib.sha256(json.dumps(cols, sort_keys=True).encode()).hexdigest()


@pytest.mark.parametrize("entry", range(len(golden("pools.json"))))
def test_reference_pool_enumeration(entry):
    e = golden("pools.json")[entry]
    E, N, K = _geom_ENK(e["geom"])
    elem = 2 if e["hw"] == "b200" else 1
    pool = R.reference_pool(E, N, K, elem=elem)
    assert len(pool) == e["size"]
    cols = {k: [int(c[k]) for c in pool] for k in ("bm", "bn", "wn", "stg", "ttn", "group_m", "split_k")}
    assert _digest(cols) == e["digest"]
    _, _, _, gm, sk = R.region(E, N, K)
    assert (gm, sk) == (e["group_m_required"], e["split_k_eligible"])


def test_grids_match_reference():
    for e in golden("grids.json"):
        E, N, K = _geom_ENK(e["geom"])
        pool = R.reference_pool(E, N, K, elem=2 if e["hw"] == "b200" else 1)
        got = [R.grid(e["counts"], c["bm"], c["ttn"], c["split_k"], N) for c in pool]
        assert got == e["grids"]


@pytest.mark.parametrize("entry", range(3))
def test_select_matches_reference(entry):
    tab = golden("tables.json")[entry]
    E, N, K = _geom_ENK(tab["geom"])
    pool = R.reference_pool(E, N, K, elem=2 if tab["hw"] == "b200" else 1)
    kappa_ok = K / 128 >= 48
    for pick in tab["picks"]:
        sel, kept = R.select(pool, tab["coeffs"], pick["counts"], N, tab["sm_count"], kappa_ok)
        assert (sel, kept) == (pick["selected"], pick["evaluations"])
    pr = tab["predict"]
    want = np.array([float.fromhex(h) for h in pr["pred"]])
    got = np.array([R.predict(*tab["coeffs"][i][:4], pr["grids"][i], tab["sm_count"]) for i in range(len(pool))])
    np.testing.assert_allclose(got, want, rtol=5e-16, atol=0)


@pytest.mark.parametrize("entry", range(3))
def test_vectorised_select_matches_reference(entry):
    """select_np (the timed CPU dispatch baseline) picks what ramp.select_config
    picked, with the same evaluation count, on the reference's fitted tables."""
    tab = golden("tables.json")[entry]
    E, N, K = _geom_ENK(tab["geom"])
    pool = R.reference_pool(E, N, K, elem=2 if tab["hw"] == "b200" else 1)
    co = np.array([c[:4] for c in tab["coeffs"]], dtype=np.float64)
    cols = {k: np.array([c[k] for c in pool]) for k in ("bm", "ttn", "split_k")}
    for pick in tab["picks"]:
        got = R.select_np(cols["bm"], cols["ttn"], cols["split_k"], co[:, 0], co[:, 1], co[:, 2], co[:, 3],
                          pick["counts"], N, tab["sm_count"], K / 128 >= 48)
        assert got == (pick["selected"], pick["evaluations"])


def test_fit_matches_reference():
    for f in golden("fits.json"):
        got = R.fit(f["g"], f["t"], 132, f["variant"])
        for key in ("a", "b", "c", "d"):
            assert got[key] == pytest.approx(f[key], rel=1e-9, abs=1e-9), (f["case"], f["variant"], key)
        assert got["uses_log"] == f["uses_log"]
        assert got["flag"] == f["condition_flag"]
        assert got["median"] == f["median_grid"]


def test_simulator_matches_reference():
    ev = golden("eval.json")
    E, N, K = _geom_ENK("OLMoE")
    pool = R.reference_pool(E, N, K)
    rr = R.round_robin(E, 64 * 8)
    quiet = dict(R.SIM_DEFAULTS, noise_cv=0.0)
    np.testing.assert_allclose(R.sim_pool_times(pool, rr, N, K, quiet, 0),
                               [float.fromhex(h) for h in ev["sim_quiet_rr64"]], rtol=1e-13)
    noisy = R.sim_pool_times(pool, rr, N, K, R.SIM_DEFAULTS, R.derive_seed(42, 2, 64, 1000, 0))
    np.testing.assert_allclose(noisy, [float.fromhex(h) for h in ev["sim_noisy_rr64"]], rtol=1e-13)
