"""One DeepSeek-V3 expert-parallel layer at world 1 through the real exchange
(ramp_ep_dispatch -> FP8 megakernel -> ramp_ep_combine), a few times: the
ncu target for the exchange's kernel breakdown (pack, NCCL send/recv,
megakernel, reduce).

    ncu --metrics gpu__time_duration.sum --csv --log-file gpurun_out/ep_launches.csv python scripts/ep_point.py
"""
import socket
import sys
from pathlib import Path

import torch
import torch.distributed as dist

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
from paper_2604_26039_b200 import ep  # noqa: E402
from paper_2604_26039_b200.catalog import BASELINE_MODELS, MoeGeometry  # noqa: E402
from paper_2604_26039_b200.config_space import HardwareModel, enumerate_b200_configs  # noqa: E402
from paper_2604_26039_b200.cost_model import active_ids_of, parse_coeff_store, read_coeff_store  # noqa: E402
from paper_2604_26039_b200.dispatch import DispatchTable, derive_seed  # noqa: E402
from paper_2604_26039_b200.routing import sample_histogram  # noqa: E402
from paper_2604_26039_b200.sweep import make_fp8_weights, make_inputs  # noqa: E402

sk = socket.socket()
sk.bind(("127.0.0.1", 0))
port = sk.getsockname()[1]
sk.close()
dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                        device_id=torch.device("cuda", 0))
geom = BASELINE_MODELS[bench.EP_MODEL]
lgeom = MoeGeometry(name="DeepSeek-V3-EP1", E=geom.E, N=geom.N, K=geom.K, top_k=geom.top_k)
pool = enumerate_b200_configs(lgeom, HardwareModel.b200(), dtype="fp8")
store = read_coeff_store(ROOT / "paper_2604_26039_b200" / "data" / f"coeffs_{bench.EP_LOCAL}_b200_fp8.json")
_, sm, co = parse_coeff_store(store)
dtab = DispatchTable(model=lgeom.name, pool=pool, coefficients=co, sm_count=sm,
                     active=active_ids_of(store)).device_table()
weights = make_fp8_weights(lgeom, seed=1000)
hs = derive_seed(42, 9, bench.EP_TOKENS, round(bench.EP_BETA * 1000), 0)
hist = sample_histogram(geom.E, bench.EP_TOKENS, geom.top_k, bench.EP_BETA, hs).histogram
x, ids, w = make_inputs(geom, hist, hs)
wcache = {}
local_fn = ep.make_local_megakernel(weights, dtab, workspace_cache=wcache)
comm = ep.EPComm()
for _ in range(3):
    out = ep.ep_moe_layer(x, ids, w, geom.E, local_fn, wire="fp8", comm=comm)
torch.cuda.synchronize()
sel = [dtab.pool_id(int(v.sel[0].item())) for v in wcache.values()]
print("ep layer ok", out.float().abs().mean().item(), "active", hist.active_experts,
      "cfg", [pool.by_id(c).to_dict() for c in sel])
comm.close()
dist.destroy_process_group()
