"""Python host mirror of the averaging round (one object per rank/GPU).

    rnd = AveragingRound(n, tensor_sizes, wire="fp16", rank=r, world=w)
    rnd.assign(fractions, sample_counts)      # LP fractions -> part offsets
    rnd.run([grad], p, m, v, step)             # one butterfly round + LAMB

`fractions` are StrategyAssignment::fractions from solve_strategy
(/root/reference/proj/src/strategy.cpp:473-498); `sample_counts` are the
weights of groups::run_plan (/root/reference/proj/include/swarmplan/groups.hpp:35-37).
Tensors are torch CUDA tensors; only their data pointers cross into
libsp_round.so (the C-ABI in include/sp_round.h). torch is plumbing here:
device memory, streams and, for world > 1, the handle all-gather.
"""
from __future__ import annotations

import ctypes
import math
from typing import Sequence

from . import _native as nat


def part_offsets(n: int, fractions: Sequence[float], align: int) -> list[int]:
    """Contiguous parts in peer order, proportional to `fractions`, every inner
    boundary a multiple of `align` (so no q8 block straddles two owners).
    offsets[k] = clamp(align * round(n * sum_{i<k} f_i / align), offsets[k-1], n).
    The paper only says 'proportional';
    the reference never materializes parts."""
    G = len(fractions)
    if G < 1:
        raise ValueError("need at least one peer")
    if any(not (f >= 0.0) or not math.isfinite(f) for f in fractions):
        raise ValueError("fractions must be finite and non-negative")
    if align < 1:
        raise ValueError("align must be positive")
    out = [0] * (G + 1)
    cum = 0.0
    for k in range(1, G):
        cum += float(fractions[k - 1])
        x = n * cum / align
        # std::llround (half away from zero) as the C++ partition.cpp does;
        # x >= 0, and x - floor(x) is exact, unlike floor(x + 0.5) (which
        # rounds 0.49999999999999994 up)
        f = math.floor(x)
        o = align * (int(f) + (1 if x - f >= 0.5 else 0))
        out[k] = min(n, max(out[k - 1], o))
    out[G] = n
    return out


class AveragingRound:
    def __init__(self, n: int, tensor_sizes: Sequence[int] | None = None, *, wire: str = "fp16",
                 q8_block: int = 4096, peers_per_rank: int = 1, rank: int = 0, world: int = 1,
                 device: int | None = None, lr: float = 1.76e-3, betas=(0.9, 0.999),
                 eps: float = 1e-6, weight_decay: float = 0.01, bias_correction: bool = True,
                 barrier_timeout_s: float = 20.0, process_group=None, shard_lamb: bool = False):
        import torch

        if wire not in nat.WIRE_FORMATS:
            raise ValueError(f"wire must be one of {sorted(nat.WIRE_FORMATS)}")
        self.n = int(n)
        self.tensor_sizes = [int(s) for s in (tensor_sizes or [n])]
        self.wire = wire
        self.q8_block = int(q8_block)
        self.L = int(peers_per_rank)
        self.rank, self.world = int(rank), int(world)
        self.G = self.L * self.world
        self.device = torch.cuda.current_device() if device is None else int(device)
        self._sizes = (ctypes.c_int64 * len(self.tensor_sizes))(*self.tensor_sizes)
        cfg = nat.SpRoundCfg(
            device=self.device, rank=self.rank, world=self.world, peers_per_rank=self.L,
            n=self.n, wire=nat.WIRE_FORMATS[wire], q8_block=self.q8_block,
            num_tensors=len(self.tensor_sizes), tensor_sizes=self._sizes, lr=lr,
            beta1=betas[0], beta2=betas[1], eps=eps, weight_decay=weight_decay,
            bias_correction=int(bool(bias_correction)), barrier_timeout_s=barrier_timeout_s,
            shard_lamb=int(bool(shard_lamb)))
        self.shard_lamb = bool(shard_lamb)
        self._lib = nat.lib()
        self._h = ctypes.c_void_p()
        nat.check(self._lib.sp_round_create(ctypes.byref(cfg), ctypes.byref(self._h)))
        self.offsets: list[int] | None = None
        self.weights: list[float] | None = None
        if self.world > 1:
            self._connect(process_group)
        self._group = process_group

    # -- multi-rank wiring ------------------------------------------------
    def _connect(self, group) -> None:
        import torch
        import torch.distributed as dist

        from .dist import exchange_handles

        nb = self._lib.sp_round_handle_bytes()
        mine = (ctypes.c_char * nb)()
        nat.check(self._lib.sp_round_export(self._h, mine))
        blob = exchange_handles(bytes(mine), group)
        buf = (ctypes.c_char * len(blob)).from_buffer_copy(blob)
        nat.check(self._lib.sp_round_connect(self._h, buf))
        dist.barrier(group=group)
        torch.cuda.synchronize(self.device)

    # -- assignment ---------------------------------------------------------
    @property
    def align(self) -> int:
        return int(self._lib.sp_round_align(self._h))

    def set_assignment(self, offsets: Sequence[int], weights: Sequence[float]) -> None:
        if len(offsets) != self.G + 1 or len(weights) != self.G:
            raise ValueError(f"need {self.G + 1} offsets and {self.G} weights")
        o = (ctypes.c_int64 * (self.G + 1))(*[int(x) for x in offsets])
        w = (ctypes.c_double * self.G)(*[float(x) for x in weights])
        nat.check(self._lib.sp_round_set_assignment(self._h, o, w))
        self.offsets, self.weights = list(map(int, offsets)), list(map(float, weights))
        if self.world > 1:
            from .dist import check_same_plan

            check_same_plan(self.offsets, self.weights, getattr(self, "_group", None))

    def assign(self, fractions: Sequence[float], weights: Sequence[float]) -> list[int]:
        offs = part_offsets(self.n, fractions, self.align)
        self.set_assignment(offs, weights)
        return offs

    # -- the round ----------------------------------------------------------
    def _st(self, stream):
        """cudaStream_t for the C-ABI: the given stream, else torch's current
        stream on this device, so the round is ordered after the caller's
        backward pass and before its next forward (the library never picks
        a stream of its own; include/sp_round.h "Streams")."""
        if stream is None:
            import torch

            return torch.cuda.current_stream(self.device).cuda_stream or None
        return (stream or None) if isinstance(stream, int) else (stream.cuda_stream or None)

    def _ptrs(self, grads):
        if len(grads) != self.L:
            raise ValueError(f"expected {self.L} local gradients")
        arr = (ctypes.c_void_p * self.L)()
        for i, g in enumerate(grads):
            arr[i] = None if g is None else self._dptr(g, self.n)
        return arr

    def _dptr(self, t, n):
        import torch

        if isinstance(t, int):
            return t
        if not (t.is_cuda and t.dtype == torch.float32 and t.is_contiguous() and t.numel() >= n):
            raise ValueError("expected a contiguous CUDA float32 tensor of at least n elements")
        return t.data_ptr()

    def run(self, grads, p, m, v, step: int, stream=None) -> None:
        st = self._st(stream)
        nat.check(self._lib.sp_round_run(self._h, self._ptrs(grads), self._dptr(p, self.n),
                                         self._dptr(m, self.n), self._dptr(v, self.n),
                                         int(step), st))

    def run_host(self, host_grads, p, m, v, step: int, stream=None, p_out=None) -> None:
        """One round from HOST gradients (sp_round_run_host): pinned CPU
        float32 tensors, copied to a double-buffered device staging area on
        the round's copy stream, so this step's copy overlaps the previous
        round. p, m, v stay device tensors. `p_out` (pinned CPU float32 of n
        elements) receives the updated parameters, copied after the round on
        `stream` (sp_round_run_host_params)."""
        import torch

        if len(host_grads) != self.L:
            raise ValueError(f"expected {self.L} local gradients")
        arr = (ctypes.c_void_p * self.L)()
        for i, g in enumerate(host_grads):
            if g is None:
                continue
            if g.is_cuda or g.dtype != torch.float32 or not g.is_contiguous() or g.numel() < self.n:
                raise ValueError("host_grads: contiguous CPU float32 tensors of at least n elements")
            arr[i] = g.data_ptr()
        out = None
        if p_out is not None:
            if (p_out.is_cuda or p_out.dtype != torch.float32 or not p_out.is_contiguous()
                    or p_out.numel() < self.n):
                raise ValueError("p_out: contiguous CPU float32 tensor of at least n elements")
            out = p_out.data_ptr()
        nat.check(self._lib.sp_round_run_host_params(self._h, arr, self._dptr(p, self.n),
                                                     self._dptr(m, self.n), self._dptr(v, self.n),
                                                     int(step), out, self._st(stream)))

    def run_phased(self, grads, p, m, v, step: int, stream=None) -> dict:
        st = self._st(stream)
        t = nat.SpPhaseTimes()
        nat.check(self._lib.sp_round_run_phased(self._h, self._ptrs(grads), self._dptr(p, self.n),
                                                self._dptr(m, self.n), self._dptr(v, self.n),
                                                int(step), st, ctypes.byref(t)))
        return {k: float(getattr(t, k)) for k, _ in nat.SpPhaseTimes._fields_}

    # -- device-side accumulation (round step 1) ---------------------------
    def accumulate(self, local_peer: int, grad, samples: float, buf: int = 0, stream=None) -> None:
        """acc[buf][local_peer] (+)= grad (fp32, device) and count `samples`."""
        st = self._st(stream)
        nat.check(self._lib.sp_round_accumulate(self._h, buf, local_peer, self._dptr(grad, self.n),
                                                float(samples), st))

    def accumulator(self, local_peer: int = 0, buf: int = 0):
        """The accumulator as a torch tensor (zero-copy view of executor memory)."""
        import torch

        ptr = self._lib.sp_round_accumulator_ptr(self._h, buf, local_peer)
        if not ptr:
            raise RuntimeError(nat.lib().sp_last_error().decode())

        class _View:  # __cuda_array_interface__ v3
            __cuda_array_interface__ = {"shape": (self.n,), "typestr": "<f4",
                                        "data": (int(ptr), False), "version": 3}

        return torch.as_tensor(_View(), device=f"cuda:{self.device}")

    def param_buffer(self):
        """shard_lamb: the flat fp32[n] parameter vector the round updates (a
        zero-copy torch view of executor memory; pass it as `p`). Owners store
        their updated ranges into every rank's copy."""
        import torch

        ptr = self._lib.sp_round_param_ptr(self._h)
        if not ptr:
            raise RuntimeError("param_buffer() needs shard_lamb=True")

        class _View:  # __cuda_array_interface__ v3
            __cuda_array_interface__ = {"shape": (self.n,), "typestr": "<f4",
                                        "data": (int(ptr), False), "version": 3}

        return torch.as_tensor(_View(), device=f"cuda:{self.device}")

    def lamb_chunks(self) -> tuple:
        """(chunks, tile) of the LAMB plan (sp_round_lamb_chunks)."""
        tile = ctypes.c_int(0)
        n = int(self._lib.sp_round_lamb_chunks(self._h, ctypes.byref(tile)))
        return n, tile.value

    def own_range(self) -> tuple[int, int]:
        """[lo, hi) of the flattened vector this rank owns (averages, and with
        shard_lamb also steps)."""
        if self.offsets is None:
            raise RuntimeError("assign() first")
        return self.offsets[self.rank * self.L], self.offsets[(self.rank + 1) * self.L]

    def add_samples(self, local_peer: int, samples: float, buf: int = 0) -> None:
        nat.check(self._lib.sp_round_add_samples(self._h, buf, local_peer, float(samples)))

    def samples(self, local_peer: int = 0, buf: int = 0) -> float:
        return float(self._lib.sp_round_samples(self._h, buf, local_peer))

    def run_accumulated(self, p, m, v, step: int, buf: int = 0, stream=None) -> None:
        """Round over the accumulators of `buf`, weighted by their sample counts.

        DPU (delayed parameter updates): step s+1 may
        accumulate into the other buffer on another stream while this round
        runs; order that stream after the round that last read the buffer it
        writes (an event recorded after run_accumulated(..., buf=b))."""
        st = self._st(stream)
        nat.check(self._lib.sp_round_run_accumulated(self._h, buf, self._dptr(p, self.n),
                                                     self._dptr(m, self.n), self._dptr(v, self.n),
                                                     int(step), st))

    # -- buffers ------------------------------------------------------------
    def wire_ptr(self, local_peer: int = 0) -> int:
        return int(self._lib.sp_round_wire_ptr(self._h, local_peer))

    @property
    def padded_n(self) -> int:
        return int(self._lib.sp_round_padded_n(self._h))

    def read(self, which: int, nbytes: int, local_peer: int = 0, offset: int = 0) -> bytes:
        buf = (ctypes.c_char * nbytes)()
        nat.check(self._lib.sp_round_read(self._h, which, local_peer, offset, buf, nbytes))
        return bytes(buf)

    def copy_trust_async(self, dst_ptr: int, stream=None) -> None:
        """Stream-ordered copy of the per-tensor trust ratios to dst_ptr
        (pinned host or device memory)."""
        st = self._st(stream)
        nat.check(self._lib.sp_round_copy_trust(self._h, dst_ptr, st))

    def read_trust(self):
        import numpy as np

        b = self.read(nat.SP_BUF_TRUST, 4 * len(self.tensor_sizes))
        return np.frombuffer(b, dtype=np.float32).copy()

    def read_wire(self, which: int = nat.SP_BUF_AVG, local_peer: int = 0):
        """(values, scales) of a wire/avg buffer as numpy arrays of length n."""
        import numpy as np

        n = self.n
        if self.wire == "fp32":
            return np.frombuffer(self.read(which, 4 * n, local_peer), np.float32).copy(), None
        if self.wire == "fp16":
            return np.frombuffer(self.read(which, 2 * n, local_peer), np.uint16).copy(), None
        nb = (n + self.q8_block - 1) // self.q8_block
        codes = np.frombuffer(self.read(which, n, local_peer), np.int8).copy()
        scales = np.frombuffer(self.read(which, 4 * nb, local_peer, offset=self.padded_n),
                               np.float32).copy()
        return codes, scales

    def close(self) -> None:
        if getattr(self, "_h", None) and self._h.value:
            self._lib.sp_round_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def fill_synthetic(t, seed: int, peer: int, scale: float, outlier_every: int = 997,
                   outlier_mult: float = 100.0, stream=None) -> None:
    """Device twin of oracle sp_oracle_fill_synthetic (bit-identical)."""
    import torch

    st = (torch.cuda.current_stream(t.device).cuda_stream if stream is None else stream.cuda_stream) or None
    nat.check(nat.lib().sp_fill_synthetic(t.data_ptr(), t.numel(), seed, peer, scale,
                                          outlier_every, outlier_mult, st))
