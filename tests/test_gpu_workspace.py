"""GPU tests (-m gpu) of the caller-managed workspace entries: mstrsm_*_ex_ws with
mstrsm_workspace_size bytes gives the library-allocating entry's results bit for bit; a
workspace that is too small or misaligned is rejected before any work is enqueued."""
import numpy as np
import pytest

from paper_1607_01477_b200 import inputs
from tests.gpu_util import dev, host

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ms():
    import torch
    assert torch.cuda.is_available(), "gpu tests need a GPU"
    import paper_1607_01477_b200 as m
    m.load()
    return m


@pytest.mark.parametrize("cplx", [False, True])
@pytest.mark.parametrize("op", [0, 1])
def test_workspace_entry_is_bitwise_the_allocating_entry(ms, cplx, op):
    import torch
    m, n, nb = 333, 70, 64
    rng = np.random.default_rng([71, op, cplx])
    U = np.triu(rng.standard_normal((m, m)) + (1j * rng.standard_normal((m, m)) if cplx else 0)) * 3.0
    U[np.arange(m), np.arange(m)] = rng.uniform(-1e-2, 1e-2, m)         # growth: rescaling on
    s = inputs.random_shifts(n, cplx, 5, radius=1e-2)
    B = inputs.random_rhs(m, n, cplx, 6)
    Ud, sd = dev(np.asfortranarray(U)), dev(np.ascontiguousarray(s))
    B1, B2 = dev(B), dev(B)
    sc1, sc2 = (torch.empty(n, dtype=torch.float64, device="cuda") for _ in range(2))
    e1, e2 = (torch.empty(n, dtype=torch.int32, device="cuda") for _ in range(2))
    f_ex = ms.mstrsm_z_ex if cplx else ms.mstrsm_d_ex
    f_ws = ms.mstrsm_z_ex_ws if cplx else ms.mstrsm_d_ex_ws
    f_ex(1, op, Ud, m, m, sd, 1, B1, m, n, None, sc1, e1, nb)
    nbytes = ms.mstrsm_workspace_size(m, n, nb, cplx, True)
    ws = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    f_ws(1, op, Ud, m, m, sd, 1, B2, m, n, None, sc2, e2, nb, ws, nbytes)
    torch.cuda.synchronize()
    assert (host(e1) < 0).any()
    assert np.array_equal(host(B1), host(B2)) and np.array_equal(host(e1), host(e2))
    with pytest.raises(ms.MstrsmError):
        f_ws(1, op, Ud, m, m, sd, 1, B2, m, n, None, sc2, e2, nb, ws, 4096)          # too small: -16
    with pytest.raises(ms.MstrsmError):
        f_ws(1, op, Ud, m, m, sd, 1, B2, m, n, None, sc2, e2, nb, ws[8:], nbytes - 8)  # misaligned: -15
