"""Per-stage CUDA-graph timings of one DeepSeek-V3 expert-parallel layer at
world 1 (the bench EP leg's workload): pack kernel alone, dispatch (pack +
NCCL), the local megakernel on the received rows, combine (NCCL + reduce)
and the whole layer -- each a graph of 4 back-to-back calls, median of 20
replays.  Shows where the exchange overhead of the bench's EP leg goes.

    python scripts/ep_breakdown.py
"""
import socket
import sys
from pathlib import Path

import numpy as np
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
store = read_coeff_store(ROOT / "paper_2604_26039_b200" / "data" / f"coeffs_{bench.EP_MODEL}_b200_fp8.json")
_, sm, co = parse_coeff_store(store)
dtab = DispatchTable(model=lgeom.name, pool=pool, coefficients=co, sm_count=sm,
                     active=active_ids_of(store)).device_table()
weights = make_fp8_weights(lgeom, seed=1000)
hs = derive_seed(42, 9, bench.EP_TOKENS, round(bench.EP_BETA * 1000), 0)
hist = sample_histogram(geom.E, bench.EP_TOKENS, geom.top_k, bench.EP_BETA, hs).histogram
x, ids, w = make_inputs(geom, hist, hs)
local_fn = ep.make_local_megakernel(weights, dtab)
comm = ep.EPComm()
K = ep.DeviceKernels()
side = torch.cuda.Stream()


def timed(fn, iters=20):
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        for _ in range(3):
            fn()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=side):
            for _ in range(4):
                fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(iters):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3 / 4)
    del g
    return float(np.median(ts))


plan, rx, rids, rw = ep.dispatch(x, ids, w, geom.E, wire="fp8", comm=comm)
partial = local_fn(rx, rids, rw)
res = {
    "pack": timed(lambda: K.pack(x, ids, w, geom.E, 1, x.shape[0], "fp8")),
    "dispatch (pack + NCCL)": timed(lambda: ep.dispatch(x, ids, w, geom.E, wire="fp8", comm=comm)),
    "local megakernel (route + FP8 megakernel)": timed(lambda: local_fn(rx, rids, rw)),
    "combine (NCCL + reduce)": timed(lambda: ep.combine(plan, partial, comm=comm)),
    "layer": timed(lambda: ep.ep_moe_layer(x, ids, w, geom.E, local_fn, wire="fp8", comm=comm)),
}
for k, v in res.items():
    print(f"{k:45s} {v:8.2f} us")
torch.cuda.synchronize()
comm.close()
dist.destroy_process_group()
