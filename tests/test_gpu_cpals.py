"""Device CP-ALS against the reference's cp_als (tests/golden/cpals.npz):
same initial factors (fp32-rounded), same layout parameters, fit history and
final model within fp32-MTTKRP accuracy."""
import numpy as np
import pytest

from conftest import GOLDEN
from paper_2309_09131_b200 import select_params
from paper_2309_09131_b200.cpals import CpalsConfig, cp_als, fit, normalize_factors

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["a", "b"])
def test_cp_als_tracks_reference(name):
    z = np.load(GOLDEN / "cpals.npz")
    subs, vals, dims = z[f"{name}_subs"], z[f"{name}_vals"], tuple(z[f"{name}_dims"])
    rank, iters, seed = (int(x) for x in z[f"{name}_cfg"])
    cfg = CpalsConfig(rank=rank, max_iters=iters, tol=1e-12, seed=seed, nu=2, gamma=1 << 20,
                      g_range=(16, 256), use_reference_params=True)
    res = cp_als(subs, vals, dims, cfg)
    want = z[f"{name}_fit"]
    assert res.iterations == len(want)
    np.testing.assert_allclose(res.fit_history, want, rtol=0, atol=2e-5)
    got_f = res.factors.to_numpy()
    for n in range(len(dims)):
        np.testing.assert_allclose(got_f[n], z[f"{name}_factor{n}"], rtol=0, atol=5e-4)
    np.testing.assert_allclose(res.factors.lambdas, z[f"{name}_lambdas"], rtol=1e-3)
    assert abs(fit(subs, vals, res.factors) - float(z[f"{name}_fit_fn"][0])) < 2e-5


def test_cp_als_device_params_and_normalize():
    z = np.load(GOLDEN / "cpals.npz")
    subs, vals, dims = z["a_subs"], z["a_vals"], tuple(z["a_dims"])
    res = cp_als(subs, vals, dims, CpalsConfig(rank=4, max_iters=5, tol=1e-12, seed=21))
    assert all(np.isfinite(res.fit_history)) and res.fit_history[-1] > res.fit_history[0]
    nf = normalize_factors(res.factors)
    for f in nf.factors:
        np.testing.assert_allclose(f.double().norm(dim=0).cpu().numpy(), 1.0, atol=1e-5)
