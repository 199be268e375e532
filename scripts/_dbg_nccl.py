import faulthandler, sys, os
faulthandler.dump_traceback_later(90, exit=True)
sys.path.insert(0, os.getcwd())
import torch
import tests.test_gpu_ep as T
from paper_2604_26039_b200.ep import EPComm, ep_moe_layer, make_local_megakernel
from tests._util import random_moe
import numpy as np
wire = sys.argv[1] if len(sys.argv) > 1 else "bf16"
E, k, H, I, S = 16, 4, 512, 256, 64
x, w1, w2, w, ids = random_moe(S, H, I, E, k, seed=21)
xt = torch.from_numpy(x).cuda().to(torch.bfloat16)
wt, it = torch.from_numpy(w).cuda(), torch.from_numpy(ids).cuda()
fn = make_local_megakernel((torch.from_numpy(w1).cuda().to(torch.bfloat16), torch.from_numpy(w2).cuda().to(torch.bfloat16)), T._bf16_table(E, H, I, k))
def body():
    print("init comm", flush=True)
    comm = EPComm()
    print("identity", flush=True)
    ident = ep_moe_layer(xt, it, wt, E, fn, wire=wire); torch.cuda.synchronize()
    print("tdist", flush=True)
    tdist = ep_moe_layer(xt, it, wt, E, fn, wire=wire, exchange="always"); torch.cuda.synchronize()
    print("nccl", flush=True)
    nccl = ep_moe_layer(xt, it, wt, E, fn, wire=wire, comm=comm); torch.cuda.synchronize()
    print("graph", flush=True)
    side = torch.cuda.Stream(); side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=side):
            cap_out = ep_moe_layer(xt, it, wt, E, fn, wire=wire, comm=comm)
    print("replay", flush=True)
    g.replay(); torch.cuda.synchronize()
    print("done", T._rel(tdist, nccl), T._rel(nccl, cap_out), flush=True)
    comm.close()
T._nccl_world1(body)
print("ok", flush=True)
