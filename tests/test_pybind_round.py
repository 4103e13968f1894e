"""The GPU round through the pybind11 module (the reference's
Python API extended with run_averaging_round on torch CUDA tensors) is the
same round as through the ctypes C-ABI binding, bit for bit."""
import numpy as np
import pytest

from paper_2106_10207_b200 import _swarmplan as sp

SIZES = [3, 1000, 70001, 2, 4096, 131075, 5]


def test_class_and_function_exported():
    assert hasattr(sp, "AveragingRound") and hasattr(sp, "run_averaging_round")


@pytest.mark.gpu
@pytest.mark.parametrize("wire", ["fp16", "q8"])
def test_pybind_round_equals_ctypes_round(wire):
    torch = pytest.importorskip("torch")
    from paper_2106_10207_b200 import AveragingRound, fill_synthetic

    n, G = sum(SIZES), 3
    fr, w = [0.2, 0.3, 0.5], [2.0, 1.0, 3.0]
    outs = []
    for route in ("ctypes", "pybind"):
        grads = []
        for g in range(G):
            t = torch.empty(n, device="cuda")
            fill_synthetic(t, 21, g, 1e-3)
            grads.append(t)
        p = torch.empty(n, device="cuda")
        fill_synthetic(p, 22, 0, 0.02, 0)
        m, v = torch.zeros(n, device="cuda"), torch.zeros(n, device="cuda")
        if route == "ctypes":
            r = AveragingRound(n, SIZES, wire=wire, peers_per_rank=G)
            r.assign(fr, w)
            for step in (1, 2, 3):
                r.run(grads, p, m, v, step)
            torch.cuda.synchronize()
            r.close()
        else:
            r = sp.AveragingRound(n, SIZES, wire=wire, peers_per_rank=G, device=torch.cuda.current_device())
            offs = r.assign(fr, w)
            assert offs[0] == 0 and offs[-1] == n and r.align == (4096 if wire == "q8" else 8)
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                for step in (1, 2, 3):
                    sp.run_averaging_round(r, grads, p, m, v, step)  # default: current stream
            torch.cuda.synchronize()
            with pytest.raises(ValueError):
                sp.run_averaging_round(r, grads[:2], p, m, v, 4)
            with pytest.raises(ValueError):
                sp.run_averaging_round(r, grads, p.double(), m, v, 4)
            del r
        outs.append([x.cpu().numpy().copy() for x in (p, m, v)])
    for a, b, name in zip(outs[0], outs[1], "pmv"):
        np.testing.assert_array_equal(a, b, err_msg=name)
