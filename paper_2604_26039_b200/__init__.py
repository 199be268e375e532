"""B200-native (sm_100a) RaMP fused-MoE hot path.

Mirrors the reference `ramp` package's API for the hot path (histogram,
grids, the four-parameter wave cost model, dispatch) and adds the GPU data
plane the reference only simulates: moe_align_block_size, the persistent
tcgen05 fused-MoE megakernel and the on-device dispatcher, all behind the C
ABI in include/ramp_b200.h.

`import paper_2604_26039_b200 as ramp` exposes the names of the reference's
`ramp/__init__.py:69-115` with the same signatures.  Three of them belong to
the reference's desk simulator, which this package replaces with measured
kernel time: `OracleParams`, `simulate_time` and `time_at_grid` have no
counterpart; `profile(...)` takes a timer (`sweep.MeasuredTimer`, the
megakernel on the GPU) where the reference takes simulator parameters.
The GPU entry points (`fused_moe`, `fused_moe_fp8`, `fused_moe_gating`,
`moe_align_block_size`, `dispatch_select`) load libramp_b200.so on first use.
"""

from .catalog import (  # noqa: F401
    BASELINE_MODELS,
    EXPECTED_CLASSIFICATION,
    MoeGeometry,
    RegimeReport,
    RegionVariables,
    classify_regime,
    find_model,
    load_catalog,
    region_variables,
)
from .config_space import (  # noqa: F401
    ConfigPool,
    EmptyPoolError,
    HardwareModel,
    TileConfig,
    enumerate_b200_configs,
    enumerate_configs,
    smem_usage,
)
from .cost_model import (  # noqa: F401
    CostCoefficients,
    FitReport,
    ProfilingSample,
    fit,
    predict,
    predict_batch,
    profiling_plan,
)
from .dispatch import (  # noqa: F401
    DispatchTable,
    RegretReport,
    SpeedupReport,
    StepCache,
    evaluate_regret,
    select_config,
    speedup_ra_vs_static,
    split_k_gate,
    static_best,
)
from .routing import (  # noqa: F401
    BetaUnreachableError,
    ExpertHistogram,
    RoutingSample,
    balancedness,
    grid_size,
    m_tile_counts,
    pool_grids,
    round_robin,
    sample_histogram,
    wave_utilization,
)
from .trace import TimingTrace, load_trace, profile, save_trace  # noqa: F401


def __getattr__(name):
    # the GPU side imports torch; keep `import paper_2604_26039_b200` light
    gpu = {"fused_moe", "fused_moe_fp8", "fused_moe_gating", "moe_align_block_size", "dispatch_select",
           "DeviceTable", "DeviceStepCache", "Workspace"}
    if name in gpu:
        from . import moe

        return getattr(moe, name)
    raise AttributeError(f"module {__name__!r} has no attribute {name!r}")


__version__ = "0.2.0"

__all__ = [
    "EXPECTED_CLASSIFICATION", "MoeGeometry", "RegimeReport", "RegionVariables", "classify_regime", "find_model",
    "load_catalog", "region_variables", "ConfigPool", "EmptyPoolError", "HardwareModel", "TileConfig",
    "enumerate_configs", "smem_usage", "CostCoefficients", "FitReport", "ProfilingSample", "fit", "predict",
    "profiling_plan", "DispatchTable", "RegretReport", "SpeedupReport", "StepCache", "evaluate_regret",
    "select_config", "speedup_ra_vs_static", "split_k_gate", "static_best", "TimingTrace", "load_trace", "profile",
    "save_trace", "BetaUnreachableError", "ExpertHistogram", "RoutingSample", "balancedness", "grid_size",
    "round_robin", "sample_histogram", "wave_utilization", "__version__",
    # B200 additions
    "BASELINE_MODELS", "enumerate_b200_configs", "predict_batch", "pool_grids", "m_tile_counts",
    "fused_moe", "fused_moe_fp8", "fused_moe_gating", "moe_align_block_size", "dispatch_select",
    "DeviceTable", "DeviceStepCache", "Workspace",
]
