"""GPU tests (-m gpu) of the host-buffer entries used for the end-to-end number: trevc_z_host and
the batched trevc_z_host_batch (uploads / downloads of neighbouring problems overlapping the
solve) give the device path's results bit for bit, and match the oracle (R20/R21)."""
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


@pytest.mark.parametrize("count", [1, 2, 5])
def test_host_batch_equals_single_calls_and_oracle(ms, count):
    m, nb = 520, 64
    Ts = [inputs.c5_grcar_like(m)] + [inputs.c3_trevc_complex(m) for _ in range(count - 1)]
    Ts = [np.asfortranarray(T) for T in Ts]
    Z = [np.zeros((m, m), complex, order="F") for _ in range(count)]   # lower triangle: see mstrsm.h
    S = [np.zeros(m) for _ in range(count)]
    E = [np.zeros(m, np.int32) for _ in range(count)]
    ms.trevc_z_host_batch(Ts, m, Z, S, E, nb)
    for k in range(count):
        Zs = np.zeros((m, m), complex, order="F")
        ss, es = np.zeros(m), np.zeros(m, np.int32)
        ms.trevc_z_host(Ts[k], m, Zs, ss, es, nb)
        assert np.array_equal(Z[k], Zs) and np.array_equal(S[k], ss) and np.array_equal(E[k], es)
    Zo, eo = oracle.trevc(Ts[0], nb=nb)
    assert (eo < -100).any()
    assert_parity(Z[0], E[0], Zo, eo, what="host batch c5")


def test_host_batch_rejects_bad_arguments(ms):
    m = 8
    T = np.asfortranarray(np.eye(m, dtype=complex))
    with pytest.raises(ms.MstrsmError):
        ms.trevc_z_host_batch([T], m, [np.zeros((m, m), complex, order="F")], None, None, 200)
