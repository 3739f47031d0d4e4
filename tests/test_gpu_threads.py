"""GPU tests (-m gpu) of the library's per-thread / per-device context: two host
threads driving one GPU, each on its own stream, get results bit-identical to one thread running
the same calls (the look-ahead's side stream and events, the copy streams of the host entries and
the status flag are per thread); and the host-buffer batch entry at a size that takes the
look-ahead path, with pinned buffers and distinct problems, against the oracle."""
import threading

import numpy as np
import pytest

import oracle
from paper_1607_01477_b200 import inputs
from tests.gpu_util import assert_parity

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ms():
    import torch
    assert torch.cuda.is_available(), "gpu tests need a GPU"
    import paper_1607_01477_b200 as m
    m.load()
    return m


def test_two_threads_two_streams_bit_identical(ms):
    import torch
    m = 1100                                      # >= 1024: the look-ahead (side stream) path
    Ts = [inputs.c5_grcar_like(m), inputs.c3_trevc_complex(m)]
    Td = [torch.from_numpy(np.asfortranarray(T)).cuda() for T in Ts]
    ref = []
    for T in Td:                                  # one thread, default stream
        Z, sc, e = ms.trevc(T, nb=128)
        torch.cuda.synchronize()
        ref.append((Z.cpu(), sc.cpu(), e.cpu()))
    out = [[None] * 3 for _ in range(2)]
    errs = []

    def worker(i):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                for rep in range(3):
                    Z, sc, e = ms.trevc(Td[i], nb=128)
                    s.synchronize()
                    out[i][rep] = (Z.cpu(), sc.cpu(), e.cpu())
        except Exception as ex:  # pragma: no cover - reported below
            errs.append(ex)

    th = [threading.Thread(target=worker, args=(i,)) for i in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    for i in range(2):
        for rep in range(3):
            Z, sc, e = out[i][rep]
            assert torch.equal(Z, ref[i][0]) and torch.equal(sc, ref[i][1]) and torch.equal(e, ref[i][2]), (i, rep)


def test_host_batch_pinned_lookahead_distinct_problems(ms):
    import torch
    m, nb, count = 1100, 128, 3
    gens = [inputs.c5_grcar_like, inputs.c3_trevc_complex, inputs.c5_grcar_like]
    Ts = []
    for k in range(count):
        T = gens[k](m) if k < 2 else gens[k](m) * (1.0 + 0.5j)          # three distinct problems
        pin = torch.empty((m, m), dtype=torch.complex128).pin_memory()
        Tp = pin.numpy().T                        # column-major view of pinned memory
        Tp[...] = T
        Ts.append(Tp)
    Zs = [torch.zeros((m, m), dtype=torch.complex128).pin_memory().numpy().T for _ in range(count)]
    Z_nan = np.full((m, m), np.nan + 0j, order="F")
    S = [np.zeros(m) for _ in range(count)]
    E = [np.zeros(m, np.int32) for _ in range(count)]
    ms.trevc_z_host_batch(Ts, m, Zs, S, E, nb)
    for k in range(count):
        Zo, eo = oracle.trevc(np.asfortranarray(Ts[k]), nb=nb)
        assert_parity(np.asarray(Zs[k]), E[k], Zo, eo, what=f"host batch problem {k}")
        assert np.array_equal(S[k], np.ldexp(1.0, E[k].astype(np.int64)))
    # single-problem entry: the upper triangle is written, the strictly lower one below the
    # 128-row diagonal tiles is left as passed (triangle-packed download)
    ms.trevc_z_host(np.asfortranarray(Ts[0]), m, Z_nan, None, None, nb)
    iu = np.triu_indices(m)
    assert np.array_equal(Z_nan[iu], np.asarray(Zs[0])[iu])
    r, c = np.tril_indices(m, -1)
    far = r // 128 > c // 128
    assert np.isnan(Z_nan[r[far], c[far]]).all()
    assert (Z_nan[r[~far], c[~far]] == 0).all()


def test_host_entries_reject_bad_arrays(ms):
    m = 16
    T = np.asfortranarray(np.eye(m, dtype=complex))
    with pytest.raises(ValueError):
        ms.trevc_z_host(np.ascontiguousarray(T + np.triu(np.ones((m, m)), 1)), m, np.zeros((m, m), complex, order="F"))
    with pytest.raises(TypeError):
        ms.trevc_z_host(T.real.copy(order="F"), m, np.zeros((m, m), complex, order="F"))
    with pytest.raises(ValueError):
        ms.trevc_z_host(T, m, np.zeros((m - 1, m), complex, order="F"))
    with pytest.raises(ValueError):
        ms.trevc_z_host(T, m, np.zeros((m, m), complex, order="F"), np.zeros(m - 1))
    with pytest.raises(ValueError):
        ms.trevc_z_host_batch([T, np.asfortranarray(np.eye(m + 2, dtype=complex))], m,
                              [np.zeros((m, m), complex, order="F")] * 2)
