"""Device problem generators against the numpy
generators: right-hand sides bitwise (same PCG64 stream), constant stencils
bitwise, variable-coefficient bands within a few ulp (CUDA cos/exp vs libm)."""

import numpy as np
import pytest

from paper_1604_00617_b200 import problems as P

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"])
def test_device_config_matches_numpy(name):
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    ref = P.make_config(name)
    dev = P.device_config(name)
    torch.cuda.synchronize()
    assert np.array_equal(dev.rhs.cpu().numpy(), ref.rhs)
    exact = P.CONFIGS[name]["kind"] != "varcoef"
    for got, want in zip(dev.bands, (ref.D_sub, ref.D_diag, ref.D_sup, ref.E, ref.F)):
        g = got.cpu().numpy()
        assert g.shape == want.shape
        if exact:
            assert np.array_equal(g, want)
        else:
            rel = np.max(np.abs(g - want) / np.abs(want))
            assert rel <= 1e-14, rel


def test_device_config_solves():
    """A factor + solve straight from device-generated inputs (config 2)."""
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_1604_00617_b200.solver import AcrSolver, relative_residual_gpu
    from paper_1604_00617_b200.system import Tolerance
    c = P.CONFIGS["cfg2"]
    d = P.device_config("cfg2")
    sol = AcrSolver(d.n_blocks, d.block_dim, Tolerance(c["eps"]), 1, c["leaf"])
    sol.factor(d.bands)
    u = sol.solve(d.rhs)
    rmax, _ = relative_residual_gpu(d.bands, u, d.rhs, d.n_blocks, d.block_dim)
    assert rmax < 1e-5
