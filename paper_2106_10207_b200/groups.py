"""Group all-reduce (m < n) on the GPU: groups::run_plan with
the class sums kept in HBM (/root/reference/proj/src/groups.cpp:117-161 is
the CPU original). Class bookkeeping, failure handling and the result flags
are the shared host code in csrc/host/groups.cpp; the arithmetic runs as
fp64 kernels (sp_vec_scale / sp_vec_sum / sp_vec_div in libsp_round.so) in
the same order as run_plan, so every value is bit-identical to the CPU run.
"""
from __future__ import annotations

import torch

from paper_2106_10207_b200 import _swarmplan


def run_plan_gpu(n: int, m: int, values: torch.Tensor, weights=(), failures=(),
                 out: torch.Tensor | None = None, exact: bool = False) -> dict:
    """values: (n, dim) float64 CUDA tensor, one row per peer. Returns
    run_plan's dict with "values" an (n, dim) float64 CUDA tensor. The
    default merge rule is the reference's (groups.cpp:126-151);
    exact=True is SPEC.md:240-241's (see groups::MergeRule)."""
    if values.dim() != 2 or values.shape[0] != n:
        raise ValueError("values must be (n, dim)")
    if not values.is_cuda or values.dtype != torch.float64:
        raise ValueError("values must be a float64 CUDA tensor")
    values = values.contiguous()
    if out is None:
        out = torch.empty_like(values)
    dim = values.shape[1]
    stream = torch.cuda.current_stream(values.device).cuda_stream
    with torch.cuda.device(values.device):
        res = _swarmplan.run_plan_device(
            n, m, [values[i].data_ptr() for i in range(n)], dim,
            [out[i].data_ptr() for i in range(n)], [float(w) for w in weights],
            [tuple(f) for f in failures], stream, exact)
    res["values"] = out
    return res
