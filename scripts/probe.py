"""Perf probe: time every B200 config of the OLMoE layer at a few (S, skew)
points with CUDA events.  Development tool; prints one line per point."""

from __future__ import annotations

import argparse
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2604_26039_b200 import moe as M  # noqa: E402
from paper_2604_26039_b200.catalog import MoeGeometry  # noqa: E402
from paper_2604_26039_b200.config_space import enumerate_b200_configs  # noqa: E402


def topk(S, k, E, skew, gen):
    if skew == 0:
        scores = torch.rand(S, E, generator=gen, device="cuda")
    else:
        bias = -skew * torch.arange(E, device="cuda", dtype=torch.float32)
        scores = torch.rand(S, E, generator=gen, device="cuda").log() * 0 + bias + torch.rand(
            S, E, generator=gen, device="cuda") * 3
    ids = scores.topk(k, dim=1).indices.to(torch.int32).contiguous()
    w = torch.softmax(torch.randn(S, k, generator=gen, device="cuda"), 1).contiguous()
    return ids, w


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--E", type=int, default=64)
    ap.add_argument("--H", type=int, default=2048)
    ap.add_argument("--I", type=int, default=1024)
    ap.add_argument("--k", type=int, default=8)
    ap.add_argument("--S", default="1,16,64,256,512")
    ap.add_argument("--skew", default="0,1.0")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--all", action="store_true")
    ap.add_argument("--graph", action="store_true", help="time CUDA-graph replays (no host overhead)")
    a = ap.parse_args()
    E, H, I, k = a.E, a.H, a.I, a.k
    gen = torch.Generator(device="cuda").manual_seed(0)
    w1 = (torch.randn(E, 2 * I, H, device="cuda", generator=gen) / H ** 0.5).to(torch.bfloat16)
    w2 = (torch.randn(E, H, I, device="cuda", generator=gen) / I ** 0.5).to(torch.bfloat16)
    pool = enumerate_b200_configs(MoeGeometry(name="p", E=E, N=2 * I, K=H, top_k=k))
    cols = pool.columns()
    n = len(pool)
    table = M.DeviceTable(bm=cols["bm"], ttn=cols["ttn"], stg=cols["stg"], split_k=cols["split_k"],
                          group_m=cols["group_m"].astype(np.int64), mode=cols.get("mode"), kps=cols.get("kps"), h3=cols.get("h3"), a=np.ones(n), b=np.zeros(n),
                          c=np.zeros(n), d=np.zeros(n), N=2 * I, kappa_ok=False, sm_count=148)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    print(f"pool {n} configs", flush=True)
    for S in map(int, a.S.split(",")):
        for skew in map(float, a.skew.split(",")):
            x = torch.randn(S, H, device="cuda", generator=gen).to(torch.bfloat16)
            ids, w = topk(S, k, E, skew, gen)
            active = int((torch.bincount(ids.view(-1).long(), minlength=E) > 0).sum())
            ws = M.Workspace(S, H, I, E, k)
            out = torch.empty(S, H, dtype=torch.bfloat16, device="cuda")
            res = []
            cfgs = list(pool) if a.all else [c for c in pool if c.stg in (2, 4, 8) and not c.group_m]
            for c in cfgs:
                for _ in range(2):
                    M.fused_moe(x, w1, w2, w, ids, table, c.id, out=out, workspace=ws)
                run = lambda: M.fused_moe(x, w1, w2, w, ids, table, c.id, out=out, workspace=ws)  # noqa: E731
                if a.graph:
                    g = torch.cuda.CUDAGraph()
                    s = torch.cuda.Stream()
                    s.wait_stream(torch.cuda.current_stream())
                    with torch.cuda.stream(s):
                        with torch.cuda.graph(g, stream=s):
                            run()
                    torch.cuda.current_stream().wait_stream(s)
                    run = g.replay
                    run()
                ts = []
                for _ in range(a.iters):
                    flush.zero_()
                    e0 = torch.cuda.Event(enable_timing=True)
                    e1 = torch.cuda.Event(enable_timing=True)
                    e0.record()
                    run()
                    e1.record()
                    torch.cuda.synchronize()
                    ts.append(e0.elapsed_time(e1) * 1000)
                res.append((float(np.median(ts)), c))
            res.sort(key=lambda r: r[0])
            byte = active * 3 * H * I * 2
            best_t, best_c = res[0]
            print(f"S={S:4d} skew={skew:.1f} active={active:3d} best={best_t:8.1f}us "
                  f"bm={best_c.bm} ttn={best_c.ttn} stg={best_c.stg} gm={int(best_c.group_m)} mode={best_c.mode} "
                  f"GB/s={byte / best_t / 1e3:7.0f} TF/s={6 * S * k * H * I / best_t / 1e6:6.1f} "
                  f"worst={res[-1][0]:8.1f}us", flush=True)
            for t, c in res[:6]:
                print(f"    {t:8.1f}us bm={c.bm} ttn={c.ttn} stg={c.stg} gm={int(c.group_m)} mode={c.mode}")


if __name__ == "__main__":
    t0 = time.time()
    main()
    print(f"probe done in {time.time() - t0:.1f}s")
