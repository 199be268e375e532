"""CPU oracle for the RaMP fused-MoE hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm may import this package, and only as the checker or the timed CPU
baseline.  The product package (paper_2604_26039_b200) never imports it and
has no CPU fallback.

Modules
  ramp_ref  numpy restatement of the reference control plane (histogram
            sampler, pool enumeration, grids, wave cost model, fit, dispatch,
            timing simulator, regret/speedup harness).  PINNED: checked
            against fixtures produced by the reference itself
            (tests/golden/gen_golden.py imports /root/reference read-only).
  moe_ref   fp32 fused-MoE forward and moe_align_block_size.  The reference
            has no implementation of either, so this half
            is PARITY UNPINNED by the reference: it restates the paper's
            semantics and vLLM's layout
            conventions, and its own frozen vectors (tests/golden/moe_*.npz)
            are the pin.
"""
