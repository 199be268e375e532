"""The shipped B200 traces through the reference's OWN trace loader and OLS
fit (ramp.load_trace / ramp.fit, /root/reference/pkg/src/ramp), against this
package's mirror: the timing-source plug point of SURVEY.md 8b.

The reference's CLI cannot ingest them unchanged: `ramp profile --oracle
trace:` validates the config ids against the workspace's *reference* pool
(ramp/cli.py:254-262, oracle.py:351), whereas these ids index the B200 pool
(enumerate_b200_configs).  The library calls do not have that restriction
(pool=None, or the B200 pool), which is what this test exercises.  Skipped
where /root/reference is absent (the GPU box)."""

from __future__ import annotations

import sys
from collections import defaultdict
from pathlib import Path

import numpy as np
import pytest

REF = Path("/root/reference/pkg/src")
DATA = Path(__file__).resolve().parents[1] / "paper_2604_26039_b200" / "data"
pytestmark = pytest.mark.skipif(not REF.exists(), reason="reference checkout not present")


@pytest.fixture(scope="module")
def ramp_ref():
    sys.path.insert(0, str(REF))
    try:
        import ramp  # the reference package, read-only
    finally:
        sys.path.remove(str(REF))
    return ramp


@pytest.mark.parametrize("name", ["trace_Qwen3-30B-A3B_b200_fp8.csv", "trace_DeepSeek-V3-EP8_b200_fp8.csv",
                                  "trace_OLMoE-1B-7B_b200.csv"])
def test_reference_loads_and_fits_b200_trace(ramp_ref, name):
    from paper_2604_26039_b200 import cost_model, trace
    from paper_2604_26039_b200.config_space import HardwareModel

    path = DATA / name
    ref_tr = ramp_ref.load_trace(path, pool=None)
    ours = trace.load_trace(path, pool=None)
    assert len(ref_tr.samples) == len(ours.samples) > 0
    for a, b in zip(ref_tr.samples, ours.samples):
        assert (a.config_id, a.S, a.beta_target, a.seed, a.g, a.time_us) == \
               (b.config_id, b.S, b.beta_target, b.seed, b.g, b.time_us)
    by_ref, by_ours = defaultdict(list), defaultdict(list)
    for s in ref_tr.samples:
        by_ref[s.config_id].append(s)
    for s in ours.samples:
        by_ours[s.config_id].append(s)
    hw_ref = ramp_ref.HardwareModel(sm_count=148, elem_size=2)
    hw = HardwareModel.b200()
    ids = sorted(by_ref)[:: max(1, len(by_ref) // 40)]
    for cid in ids:
        for variant in ("P2", "P3", "P4"):
            r = ramp_ref.fit(by_ref[cid], hw_ref, variant)
            o = cost_model.fit(by_ours[cid], hw, variant)
            got = np.array([o.coefficients.a, o.coefficients.b, o.coefficients.c, o.coefficients.d])
            want = np.array([r.coefficients.a, r.coefficients.b, r.coefficients.c, r.coefficients.d])
            np.testing.assert_allclose(got, want, rtol=1e-9, atol=1e-9 * max(1.0, float(np.abs(want).max())))
            assert o.coefficients.uses_log == r.coefficients.uses_log
            assert o.r_squared == pytest.approx(r.r_squared, rel=1e-9, abs=1e-12)


def test_reference_load_trace_with_b200_pool(ramp_ref):
    """ramp.load_trace validates ids against whatever pool it is given: with
    the B200 pool every id of the shipped trace is known."""
    from paper_2604_26039_b200.catalog import BASELINE_MODELS
    from paper_2604_26039_b200.config_space import HardwareModel, enumerate_b200_configs

    pool = enumerate_b200_configs(BASELINE_MODELS["Qwen3-30B-A3B"], HardwareModel.b200(), dtype="fp8")
    tr = ramp_ref.load_trace(DATA / "trace_Qwen3-30B-A3B_b200_fp8.csv", pool=pool)
    assert {s.config_id for s in tr.samples} <= {c.id for c in pool}
