"""GPU tests (-m gpu): the library's calls are stream-capturable, so a caller that repeats a solve
shape can capture it once into a CUDA graph and replay it (c1 0.183 -> 0.170 ms per
call replayed, `profiles/r02/rows_graph_r02.jsonl`).  Replays of the captured safe solve and
TriangEig reproduce the direct calls bit for bit, also after the inputs are refilled in place."""
import numpy as np
import pytest

from paper_1607_01477_b200 import inputs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ms():
    import torch
    assert torch.cuda.is_available(), "gpu tests need a GPU"
    import paper_1607_01477_b200 as m
    m.load()
    return m


def _capture(torch, fn):
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            out = fn()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    return g, out


def test_graph_replay_of_safe_solve_is_bit_identical(ms):
    import torch
    U, s, B = inputs.c1_plain_real()
    dev = lambda x: torch.from_numpy(np.asfortranarray(x)).cuda()
    Ud, sd, B0 = dev(U), dev(s), dev(B)
    X_direct, sc_direct, e_direct = ms.solve(Ud, sd, B0.clone(), safe=True, nb=32)
    Bw = B0.clone()
    ms.solve(Ud, sd, Bw, safe=True, nb=32)                  # warm-up (first-use set-up outside capture)
    g, (Xg, scg, eg) = _capture(torch, lambda: (Bw.copy_(B0), ms.solve(Ud, sd, Bw, safe=True, nb=32))[1])
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    assert torch.equal(Xg, X_direct) and torch.equal(eg, e_direct) and torch.equal(scg, sc_direct)
    # new right-hand sides written into the captured input buffer: the replay solves them
    B2 = dev(inputs.random_rhs(256, 64, False, 99))
    B0.copy_(B2)
    g.replay()
    X2, _, e2 = ms.solve(Ud, sd, B2.clone(), safe=True, nb=32)
    torch.cuda.synchronize()
    assert torch.equal(Xg, X2) and torch.equal(eg, e2)


def test_graph_replay_of_trevc_is_bit_identical(ms):
    import torch
    T = torch.from_numpy(np.asfortranarray(inputs.c3_trevc_complex(300))).cuda()
    Z1, s1, e1 = ms.trevc(T, nb=64)
    g, (Zg, sg, eg) = _capture(torch, lambda: ms.trevc(T, nb=64))
    g.replay()
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(Zg, Z1) and torch.equal(eg, e1) and torch.equal(sg, s1)
