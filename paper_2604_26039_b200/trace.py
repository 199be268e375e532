"""Timing traces and the profiling sweep -- mirror of the trace half of
ramp/oracle.py (the simulator half is replaced by measured B200 kernel times).

The trace CSV `config_id,S,beta_target,seed,grid,time_us` is the
reference's own plug point for real kernel timings (ramp/oracle.py:58,
:328-363; `ramp profile --oracle trace:<csv>`, ramp/cli.py:259-263): a trace
written here loads unchanged with `ramp.load_trace`, and vice versa.
`profile` walks the same (S, beta, rep) grid with the same seed derivation as
ramp.oracle.profile (:257-297) but asks a timer -- on the GPU, the measured
megakernel -- instead of the simulator.
"""

from __future__ import annotations

import csv
import io
from dataclasses import dataclass
from pathlib import Path

from .catalog import MoeGeometry
from .config_space import ConfigPool
from .cost_model import ProfilingSample
from .dispatch import HIST_DOMAIN, NOISE_DOMAIN, derive_seed
from .routing import pool_grids, sample_histogram

TRACE_HEADER = "config_id,S,beta_target,seed,grid,time_us"


@dataclass
class TimingTrace:
    model: str
    samples: list[ProfilingSample]
    provenance: str  # "measured" | "simulator" | "external"


def _row(s: ProfilingSample) -> str:
    return f"{s.config_id},{s.S},{s.beta_target:.6g},{s.seed},{s.g},{s.time_us:.6f}"


def save_trace(trace: TimingTrace, path: str | Path) -> None:
    Path(path).write_text("\n".join([TRACE_HEADER] + [_row(s) for s in trace.samples]) + "\n")


def write_resumable(trace: TimingTrace, path: Path) -> None:
    """Append the rows an existing file lacks after checking its prefix is
    byte-identical (ramp/oracle.py:309-325)."""
    lines = [TRACE_HEADER] + [_row(s) for s in trace.samples]
    have = [ln for ln in path.read_text().splitlines() if ln.strip()] if path.exists() else []
    if len(have) > len(lines):
        raise ValueError(f"{path}: existing trace has more rows than this run produces")
    for i, ln in enumerate(have):
        if ln != lines[i]:
            raise ValueError(f"{path}: line {i + 1} of the existing trace does not match this run "
                             "(different seed or plan?); refusing to append")
    with path.open("a") as fh:
        for ln in lines[len(have):]:
            fh.write(ln + "\n")


def load_trace(csv_path: str | Path, pool: ConfigPool | None = None) -> TimingTrace:
    """Parse and validate a trace (ramp/oracle.py:328-363): exact header, six
    fields, positive times, known ids, no duplicate (id, S, beta, seed)."""
    path = Path(csv_path)
    rows = [r for r in csv.reader(io.StringIO(path.read_text())) if r]
    if not rows:
        raise ValueError(f"{path}: empty trace")
    if ",".join(rows[0]) != TRACE_HEADER:
        raise ValueError(f"{path}: bad header; expected {TRACE_HEADER!r}")
    known = {c.id for c in pool} if pool is not None else None
    seen: set = set()
    out = []
    for lineno, r in enumerate(rows[1:], start=2):
        if len(r) != 6:
            raise ValueError(f"{path}: row {lineno}: expected 6 fields, got {len(r)}")
        try:
            cid, S, seed, g = int(r[0]), int(r[1]), int(r[3]), int(r[4])
            beta, t = float(r[2]), float(r[5])
        except ValueError as exc:
            raise ValueError(f"{path}: row {lineno}: {exc}") from exc
        if t <= 0:
            raise ValueError(f"{path}: row {lineno}: non-positive time {t}")
        if known is not None and cid not in known:
            raise ValueError(f"{path}: row {lineno}: unknown config_id {cid}")
        key = (cid, S, beta, seed)
        if key in seen:
            raise ValueError(f"{path}: row {lineno}: duplicate sample {key}")
        seen.add(key)
        out.append(ProfilingSample(config_id=cid, S=S, beta_target=beta, seed=seed, g=g, time_us=t))
    return TimingTrace(model=pool.geom.name if pool is not None else path.stem, samples=out,
                       provenance="external")


def profile(pool: ConfigPool, geom: MoeGeometry, plan: list[tuple[int, float]], timer,
            seeds_per_point: int = 3, master_seed: int = 42, trace_path: str | Path | None = None,
            provenance: str = "measured") -> TimingTrace:
    """Every config x plan point x routing seed, timed by `timer.pool_times`.
    Sample identity comes from (master seed, S, beta, rep), never execution
    order, so an interrupted sweep resumes to a byte-identical file."""
    if not plan:
        raise ValueError("profiling plan is empty")
    samples = []
    for S, beta in plan:
        mb = round(beta * 1000)
        for rep in range(seeds_per_point):
            hs = derive_seed(master_seed, HIST_DOMAIN, S, mb, rep)
            hist = sample_histogram(geom.E, S, geom.top_k, beta, hs).histogram
            ps = derive_seed(master_seed, NOISE_DOMAIN, S, mb, rep)
            grids = pool_grids(pool, hist)
            times = timer.pool_times(pool, hist, ps, grids=grids)
            for c in pool:
                samples.append(ProfilingSample(config_id=c.id, S=S, beta_target=beta, seed=hs,
                                               g=int(grids[c.id]), time_us=round(float(times[c.id]), 6)))
    trace = TimingTrace(model=geom.name, samples=samples, provenance=provenance)
    if trace_path is not None:
        write_resumable(trace, Path(trace_path))
    return trace
