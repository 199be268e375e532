"""The product's host-side mirror of the reference API (paper_2604_26039_b200)
against the reference's own outputs and the oracle -- CPU only.

The regret / speedup harness is checked by feeding it the oracle's
restatement of the reference simulator and the oracle's selector: it must
reproduce the reference's CSV reports byte for byte (tests/golden/eval.json).
"""

from __future__ import annotations

import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

from oracle import ramp_ref as R
from paper_2604_26039_b200 import catalog as C
from paper_2604_26039_b200 import config_space as CS
from paper_2604_26039_b200 import cost_model as CM
from paper_2604_26039_b200 import dispatch as D
from paper_2604_26039_b200 import routing as RT
from paper_2604_26039_b200 import trace as T
from tests._util import GEOMS, golden
from tests.test_oracle_golden import _geom_ENK


def _geom(name):
    E, N, K = _geom_ENK(name)
    k = GEOMS.get(name, {}).get("top_k", 8)
    return C.MoeGeometry(name=name, E=E, N=N, K=K, top_k=k)


def test_sampler_and_balancedness_bit_exact():
    for s in golden("histograms.json")["samples"]:
        if "unreachable" in s:
            with pytest.raises(RT.BetaUnreachableError):
                RT.sample_histogram(s["E"], s["S"], s["top_k"], s["beta"], int(s["seed"]))
            continue
        smp = RT.sample_histogram(s["E"], s["S"], s["top_k"], s["beta"], int(s["seed"]))
        assert list(smp.histogram.counts) == s["counts"]
        assert smp.beta_achieved == pytest.approx(s["beta_achieved"], rel=1e-12, abs=1e-12)
    for row in golden("histograms.json")["balancedness"]:
        assert RT.balancedness(RT.ExpertHistogram(tuple(row["counts"]))) == pytest.approx(row["beta"], rel=1e-12)


def test_sampler_argument_errors():
    with pytest.raises(ValueError, match="S must be"):
        RT.sample_histogram(4, 0, 2, 0.5, 0)
    with pytest.raises(ValueError, match="top_k must be"):
        RT.sample_histogram(4, 8, 0, 0.5, 0)
    with pytest.raises(ValueError, match="beta_target must be"):
        RT.sample_histogram(4, 8, 2, 1.5, 0)
    with pytest.raises(RT.BetaUnreachableError, match="E=1"):
        RT.sample_histogram(1, 8, 2, 0.5, 0)


@pytest.mark.parametrize("entry", range(len(golden("pools.json"))))
def test_reference_pool_mirror(entry):
    e = golden("pools.json")[entry]
    g = _geom(e["geom"])
    hw = CS.HardwareModel.b200() if e["hw"] == "b200" else CS.HardwareModel()
    pool = CS.enumerate_configs(g, hw, C.classify_regime(C.region_variables(g)))
    cols = {k: [int(getattr(c, k)) for c in pool] for k in ("bm", "bn", "wn", "stg", "ttn", "group_m", "split_k")}
    assert len(pool) == e["size"]
    assert hashlib.sha256(json.dumps(cols, sort_keys=True).encode()).hexdigest() == e["digest"]


def test_catalog_classification():
    for g in C.load_catalog():
        v = C.region_variables(g)
        rep = C.classify_regime(v)
        rho, lam, kappa, regime, modes = C.EXPECTED_CLASSIFICATION[g.name]
        assert (int(v.rho), v.lam, int(v.kappa), rep.regime, rep.predicted_modes) == (rho, lam, kappa, regime, modes)


def test_pool_grids_mirror():
    for e in golden("grids.json"):
        g = _geom(e["geom"])
        hw = CS.HardwareModel.b200() if e["hw"] == "b200" else CS.HardwareModel()
        pool = CS.enumerate_configs(g, hw, C.classify_regime(C.region_variables(g)))
        hist = RT.ExpertHistogram(tuple(e["counts"]))
        assert RT.pool_grids(pool, hist).tolist() == e["grids"]
        for cfg in list(pool)[::97]:
            assert RT.grid_size(cfg, hist, g) == e["grids"][cfg.id]


def test_fit_mirror():
    for f in golden("fits.json"):
        samples = [CM.ProfilingSample(config_id=0, S=8, beta_target=0.5, seed=i, g=g, time_us=t)
                   for i, (g, t) in enumerate(zip(f["g"], f["t"]))]
        rep = CM.fit(samples, CS.HardwareModel(), f["variant"])
        co = rep.coefficients
        for key in ("a", "b", "c", "d"):
            assert getattr(co, key) == pytest.approx(f[key], rel=1e-9, abs=1e-9)
        assert co.uses_log == f["uses_log"]
        assert rep.condition_flag == f["condition_flag"]
        assert rep.r_squared == pytest.approx(f["r_squared"], rel=1e-9, abs=1e-12)


def test_predict_scalar_and_batch():
    co = CM.CostCoefficients(a=10.0, b=3.0, c=0.25, d=1.5, uses_log=True, variant="P4")
    hw = CS.HardwareModel()
    assert CM.predict(co, 100, hw) == pytest.approx(10 + 3 + 25 + 1.5 * np.log(101))
    got = CM.predict_batch(np.array([10.0]), np.array([3.0]), np.array([0.25]), np.array([1.5]), [100], 132)
    assert got[0] == pytest.approx(10 + 3 + 25 + 1.5 * np.log(101))


def test_step_cache_contract():
    cache = D.StepCache()
    cache.advance(0)
    cache.selection[64] = 5
    cache.advance(0)
    assert cache.selection == {64: 5}
    cache.advance(1)
    assert cache.selection == {}


def test_plans_and_test_points():
    g = _geom("OLMoE")
    assert CM.profiling_plan(g) == [tuple(p) for p in CM.profiling_plan(g)]
    assert [list(p) for p in D.default_test_points(g)] == golden("eval.json")["default_test_points"]


class OracleTimer:
    """The reference simulator (via the oracle restatement) behind the
    product's timer interface."""

    def __init__(self, pool, geom, params):
        self.cfgs = [dict(bm=c.bm, ttn=c.ttn, stg=c.stg, group_m=c.group_m, split_k=c.split_k) for c in pool]
        self.geom, self.params = geom, params

    def quiet(self):
        return OracleTimer.__new__(OracleTimer).__init_from(self)

    def __init_from(self, other):
        self.cfgs, self.geom = other.cfgs, other.geom
        self.params = dict(other.params, noise_cv=0.0)
        return self

    def pool_times(self, pool, hist, point_seed, shared_noise=False, grids=None):
        return R.sim_pool_times(self.cfgs, list(hist.counts), self.geom.N, self.geom.K, self.params, point_seed,
                                shared_noise=shared_noise)


def _olmoe_table():
    g = _geom("OLMoE")
    pool = CS.enumerate_configs(g, CS.HardwareModel(), C.classify_regime(C.region_variables(g)))
    tab = golden("tables.json")[0]
    coeffs = {i: CM.CostCoefficients(a=c[0], b=c[1], c=c[2], d=c[3], uses_log=bool(c[4]), variant="P4")
              for i, c in enumerate(tab["coeffs"])}
    table = D.DispatchTable(model="OLMoE", pool=pool, coefficients=coeffs, sm_count=132)
    coeff_list = tab["coeffs"]
    cfgs = [dict(bm=c.bm, ttn=c.ttn, split_k=c.split_k) for c in pool]

    def selector(_, hist):
        return R.select(cfgs, coeff_list, list(hist.counts), g.N, 132, False)[0]

    return g, pool, table, selector


def test_regret_and_speedup_harness_reproduce_reference_reports():
    g, pool, table, selector = _olmoe_table()
    ev = golden("eval.json")
    timer = OracleTimer(pool, g, R.SIM_DEFAULTS)
    points = [tuple(p) for p in ev["points"]]
    reg = D.evaluate_regret(table, pool, g, timer, test_points=points, seeds_per_point=2, selector=selector)
    spd = D.speedup_ra_vs_static(table, pool, g, timer, points=points, seeds_per_point=2, selector=selector)
    assert reg.to_csv() == ev["regret_csv"]
    assert spd.to_csv() == ev["speedup_csv"]
    assert D.static_best(pool, g, timer, [8, 64]) == ev["static_best_8_64"]


def test_trace_round_trip_and_validation(tmp_path):
    g, pool, table, _ = _olmoe_table()
    timer = OracleTimer(pool, g, R.SIM_DEFAULTS)
    plan = [(8, 0.5), (32, 1.0)]
    path = tmp_path / "trace.csv"
    tr = T.profile(pool, g, plan, timer, seeds_per_point=1, trace_path=path, provenance="simulator")
    assert path.read_text().splitlines()[0] == T.TRACE_HEADER
    back = T.load_trace(path, pool)
    assert [(s.config_id, s.g, s.time_us) for s in back.samples] == [(s.config_id, s.g, s.time_us) for s in tr.samples]
    T.profile(pool, g, plan, timer, seeds_per_point=1, trace_path=path)  # resume: identical, nothing appended
    assert len(path.read_text().splitlines()) == 1 + len(tr.samples)
    bad = tmp_path / "bad.csv"
    bad.write_text(T.TRACE_HEADER + "\n0,8,0.5,1,5,-1.0\n")
    with pytest.raises(ValueError, match="non-positive"):
        T.load_trace(bad, pool)


def test_topk_from_histogram_realises_counts():
    for s in golden("histograms.json")["samples"][:60]:
        if "counts" not in s:
            continue
        ids = RT.topk_from_histogram(s["counts"], s["S"], s["top_k"], 7)
        assert ids.shape == (s["S"], s["top_k"])
        assert np.bincount(ids.ravel(), minlength=s["E"]).tolist() == s["counts"]


def test_b200_pool_is_kernel_admissible():
    for name, g in C.BASELINE_MODELS.items():
        pool = CS.enumerate_b200_configs(g)
        assert len(pool) > 0
        for c in pool:
            assert CS.b200_smem_bytes(c.bm, c.ttn, c.stg, c.mode) <= CS.B200_SMEM_LIMIT
            assert (g.N // 2) % (c.ttn // 2) == 0
        assert [c.id for c in pool] == list(range(len(pool)))


def test_phase3_chunk_variants():
    """h3 > 1 (opt-in): split-mode BF16 only, h3 <= ttn/128, d_model chunks
    divisible by h3; the job grid counts H/(128*h3) phase-3 jobs per M-tile."""
    g = C.BASELINE_MODELS["OLMoE-1B-7B"]
    base = CS.enumerate_b200_configs(g)
    ext = CS.enumerate_b200_configs(g, phase3_chunks=True)
    assert all(c.h3 == 1 for c in base)
    extra = [c for c in ext if c.h3 > 1]
    assert len(ext) == len(base) + len(extra) and extra
    cols = ext.columns()
    for c in extra:
        assert c.mode == 1 and c.dtype == "bf16" and c.h3 <= c.ttn // 128 and c.bm >= CS.B200_H3_MIN_BM
        assert cols["ntile"][c.id] == g.N // c.ttn + g.K // 128 // c.h3
        assert c.to_dict()["h3"] == c.h3
    with pytest.raises(ValueError):
        CS.TileConfig(id=0, bm=64, bn=128, wn=1, stg=3, ttn=128, family="b200", mode=1, h3=2)  # h3 > ttn/128
    with pytest.raises(ValueError):
        CS.TileConfig(id=0, bm=64, bn=128, wn=2, stg=3, ttn=256, family="b200", mode=0, h3=2)  # fused mode
    with pytest.raises(ValueError):
        CS.TileConfig(id=0, bm=64, bn=128, wn=2, stg=3, ttn=256, family="b200", mode=1, h3=3)


# ------------------------------------------------------------- B4 variant
def _b4_table(seed=0):
    from paper_2604_26039_b200.catalog import BASELINE_MODELS
    from paper_2604_26039_b200.config_space import enumerate_b200_configs
    from paper_2604_26039_b200.cost_model import CostCoefficients
    from paper_2604_26039_b200.dispatch import DispatchTable

    g = BASELINE_MODELS["OLMoE-1B-7B"]
    pool = enumerate_b200_configs(g)
    rng = np.random.default_rng(seed)
    co = {c.id: CostCoefficients(a=float(rng.uniform(10, 40)), b=float(rng.uniform(0, 20)),
                                 c=float(rng.uniform(0, 0.3)), d=float(rng.uniform(-2, 5)), uses_log=True,
                                 variant="B4", lam=float(rng.choice(np.linspace(0, 1, 21)))) for c in pool}
    return g, pool, co, DispatchTable(model="t", pool=pool, coefficients=co, sm_count=148)


def test_b4_host_select_matches_oracle():
    """The host mirror of the B4 dispatcher and the oracle restatement pick
    the same config on random histograms (the device path is held to the
    same oracle in test_gpu_kernels)."""
    from oracle import ramp_ref as R
    from paper_2604_26039_b200.routing import ExpertHistogram

    g, pool, co, table = _b4_table()
    cols = pool.columns()
    cfgs = [dict(bm=c.bm, ttn=c.ttn, split_k=c.split_k) for c in pool]
    coeffs = [[co[i].a, co[i].b, co[i].c, co[i].d] for i in range(len(pool))]
    lam = [co[i].lam for i in range(len(pool))]
    rng = np.random.default_rng(1)
    for _ in range(60):
        counts = rng.multinomial(int(rng.integers(1, 4096)), rng.dirichlet(np.full(64, 0.3)))
        want, _ = R.select(cfgs, coeffs, counts.tolist(), g.N, 148, True, ntile=cols["ntile"].tolist(),
                           omega_max=float("inf"), lam=lam)
        assert table.host_select(ExpertHistogram(tuple(int(c) for c in counts))) == want
        co4 = np.array(coeffs)
        got = R.select_np(cols["bm"], cols["ttn"], cols["split_k"], co4[:, 0], co4[:, 1], co4[:, 2], co4[:, 3],
                          counts, g.N, 148, True, ntile=cols["ntile"], omega_max=float("inf"), lam=np.array(lam))
        assert got[0] == want


def test_b4_fit_recovers_planted_model():
    from paper_2604_26039_b200.config_space import HardwareModel
    from paper_2604_26039_b200.cost_model import B4Features, ProfilingSample, fit_b4, traffic_grid

    hw = HardwareModel.b200()
    rng = np.random.default_rng(2)
    n = 60
    n_act = rng.integers(1, 65, n)
    mt = n_act + rng.integers(0, 200, n)
    jpm = 24
    g = mt * jpm
    lam = 0.35
    gl = traffic_grid(jpm, n_act, mt, lam)
    t = 20.0 + 3.0 * np.ceil(g / 148) + 0.05 * gl + 1.5 * np.log(gl + 1.0)
    samples = [ProfilingSample(config_id=0, S=8, beta_target=0.5, seed=i, g=int(g[i]), time_us=float(t[i]))
               for i in range(n)]
    feats = B4Features(g=g, n_act=n_act, m_tiles=mt, jobs_per_mtile=jpm)
    for relative in (False, True):  # B4 and B4r recover an exact model alike
        r = fit_b4(samples, feats, hw, relative=relative)
        c = r.coefficients
        assert c.variant == "B4" and abs(c.lam - lam) < 1e-9
        assert np.allclose([c.a, c.b, c.c, c.d], [20.0, 3.0, 0.05, 1.5], rtol=1e-6, atol=1e-6)
        assert r.r_squared > 1 - 1e-9


def test_b4r_weights_relative_residuals():
    """On data no model fits exactly, B4r trades absolute error on the long
    points for relative error on the short ones."""
    from paper_2604_26039_b200.config_space import HardwareModel
    from paper_2604_26039_b200.cost_model import B4Features, ProfilingSample, fit_b4, traffic_grid

    hw = HardwareModel.b200()
    rng = np.random.default_rng(3)
    n = 80
    n_act = rng.integers(1, 65, n)
    mt = n_act + rng.integers(0, 400, n)
    jpm = 24
    g = mt * jpm
    t = 20.0 + 3.0 * np.ceil(g / 148) + 0.05 * traffic_grid(jpm, n_act, mt, 0.35) + 0.002 * g ** 1.3
    samples = [ProfilingSample(config_id=0, S=8, beta_target=0.5, seed=i, g=int(g[i]), time_us=float(t[i]))
               for i in range(n)]
    feats = B4Features(g=g, n_act=n_act, m_tiles=mt, jobs_per_mtile=jpm)

    def rel_err(rep):
        c = rep.coefficients
        gl = traffic_grid(jpm, n_act, mt, c.lam)
        pred = c.a + c.b * np.ceil(g / 148) + c.c * gl + c.d * np.log(gl + 1.0)
        return np.abs(pred / t - 1.0)

    abs_fit, rel_fit = fit_b4(samples, feats, hw), fit_b4(samples, feats, hw, relative=True)
    short = t < np.median(t)
    assert np.mean(rel_err(rel_fit)[short] ** 2) <= np.mean(rel_err(abs_fit)[short] ** 2)


def test_b4_coeff_store_round_trip_and_validation():
    from paper_2604_26039_b200.cost_model import CostCoefficients, FitReport, coeff_store_dict, parse_coeff_store

    co = CostCoefficients(a=1.0, b=2.0, c=0.1, d=0.5, uses_log=True, variant="B4", lam=0.25)
    rep = FitReport(coefficients=co, r_squared=0.99, n_samples=10, median_grid=100.0, condition_flag=False)
    _, _, back = parse_coeff_store(coeff_store_dict("m", 148, {0: rep}))
    assert back[0] == co
    with pytest.raises(ValueError):
        CostCoefficients(a=1.0, b=0.0, c=0.1, d=0.0, uses_log=False, variant="P2", lam=0.5)
    with pytest.raises(ValueError):
        CostCoefficients(a=1.0, b=0.0, c=0.1, d=0.0, uses_log=True, variant="B4", lam=1.5)


def test_shipped_olmoe_coeffs_load_into_the_table():
    """The committed coefficient store matches the current B200 pool."""
    from paper_2604_26039_b200.catalog import BASELINE_MODELS
    from paper_2604_26039_b200.config_space import enumerate_b200_configs
    from paper_2604_26039_b200.cost_model import parse_coeff_store, read_coeff_store
    from paper_2604_26039_b200.dispatch import DispatchTable

    g = BASELINE_MODELS["OLMoE-1B-7B"]
    pool = enumerate_b200_configs(g)
    path = Path(__file__).resolve().parents[1] / "paper_2604_26039_b200" / "data" / "coeffs_OLMoE-1B-7B_b200.json"
    _, sm, co = parse_coeff_store(read_coeff_store(path))
    DispatchTable(model=g.name, pool=pool, coefficients=co, sm_count=sm)


def test_pruned_table_masks_and_maps_ids():
    """DispatchTable(active=...): inactive configs are never selected on the
    host, and the compacted device table maps its indices back to pool ids."""
    from paper_2604_26039_b200.catalog import BASELINE_MODELS
    from paper_2604_26039_b200.config_space import HardwareModel, enumerate_b200_configs
    from paper_2604_26039_b200.cost_model import CostCoefficients, useful_configs
    from paper_2604_26039_b200.dispatch import DispatchTable
    from paper_2604_26039_b200.routing import sample_histogram

    geom = BASELINE_MODELS["OLMoE-1B-7B"]
    pool = enumerate_b200_configs(geom, HardwareModel.b200())
    rng = np.random.default_rng(0)
    co = {c.id: CostCoefficients(a=float(rng.uniform(10, 50)), b=float(rng.uniform(0, 5)), c=0.01, d=0.5,
                                 uses_log=True, variant="P4") for c in pool}
    full = DispatchTable(model="m", pool=pool, coefficients=co, sm_count=148)
    hist = sample_histogram(geom.E, 64, geom.top_k, 0.5, 7).histogram
    best = full.host_select(hist)
    active = tuple(i for i in range(0, len(pool), 3) if i != best)
    pruned = DispatchTable(model="m", pool=pool, coefficients=co, sm_count=148, active=active)
    sel = pruned.host_select(hist)
    assert sel in active and sel != best
    p_full, p_pruned = full.host_predict(hist), pruned.host_predict(hist)
    assert np.isinf(p_pruned[best]) and p_pruned[sel] == p_full[sel]
    dt = pruned.device_table(device="cpu")
    assert len(dt) == len(active)
    assert [dt.pool_id(i) for i in range(len(dt))] == sorted(active)
    assert dt.table_index(active[5]) == 5 and dt.table_index(-1) == -1
    with pytest.raises(ValueError):
        dt.table_index(best)
    with pytest.raises(ValueError):
        DispatchTable(model="m", pool=pool, coefficients=co, sm_count=148, active=(len(pool),))

    class S:
        def __init__(self, cid, t, seed):
            self.config_id, self.time_us, self.S, self.beta_target, self.seed = cid, t, 8, 0.5, seed

    samples = [S(0, 10.0, 1), S(1, 10.4, 1), S(2, 12.0, 1), S(0, 20.0, 2), S(2, 19.0, 2)]
    assert useful_configs(samples, 0.05) == (0, 1, 2)
    assert useful_configs(samples, 0.01) == (0, 2)


def test_triton_pool_and_config_dict():
    """The third-party (vLLM Triton fused_moe) pool: grid semantics of the
    reference (g = sum ceil(c_e/BM) * ceil(N/BN)) and the override dicts."""
    from paper_2604_26039_b200.catalog import BASELINE_MODELS
    from paper_2604_26039_b200.config_space import enumerate_triton_configs, triton_config_dict
    from paper_2604_26039_b200.routing import pool_grids, sample_histogram

    geom = BASELINE_MODELS["OLMoE-1B-7B"]
    pool = enumerate_triton_configs(geom)
    assert len(pool) == 40 and all(c.family == "triton" for c in pool)
    hist = sample_histogram(geom.E, 32, geom.top_k, 0.5, 3).histogram
    counts = np.asarray(hist.counts)
    g = pool_grids(pool, hist)
    for c in pool:
        want = int(sum(-(-n // c.bm) for n in counts if n > 0)) * (-(-geom.N // c.ttn))
        assert g[c.id] == want
        d = triton_config_dict(c)
        assert (d["BLOCK_SIZE_M"], d["BLOCK_SIZE_N"], d["BLOCK_SIZE_K"]) == (c.bm, c.ttn, 64 * c.kps)
        assert d["num_stages"] * (c.bm + c.ttn) * d["BLOCK_SIZE_K"] * 2 <= 200 * 1024
