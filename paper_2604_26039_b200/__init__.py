"""B200-native (sm_100a) RaMP fused-MoE hot path.

Mirrors the reference `ramp` package's API for the hot path (histogram,
grids, the four-parameter wave cost model, dispatch) and adds the GPU data
plane the reference only simulates: moe_align_block_size, the persistent
tcgen05 fused-MoE megakernel and the on-device dispatcher, all behind the C
ABI in include/ramp_b200.h.
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

__version__ = "0.1.0"
