"""The huge-tensor path (config 5: 3.6B nonzeros): the bucketed generator
draws the same SET of nonzeros as the single-sort generator, and the lean
build produces bit-identically the plan, records and slot maps of the regular
build (so everything the parity tests prove for the regular build carries
over); a sweep on the lean-built layout is bitwise the same."""
import numpy as np
import pytest
import torch

from gpu_helpers import params_of

pytestmark = pytest.mark.gpu


def _coord_set(c: torch.Tensor) -> np.ndarray:
    c = c.to(torch.int64).cpu().numpy()
    return np.sort((c[:, 0] << 42) | (c[:, 1] << 21) | c[:, 2])


@pytest.mark.parametrize("dims,law,nnz", [
    ((46, 3000, 3000), (None, 1.0, 1.0), 400_000),     # config-5 law, small
    ((1200, 900, 2800), (1.1, 1.1, 1.1), 300_000),     # Zipf on the bucket mode
])
def test_bucketed_generator_same_set(dims, law, nnz):
    from paper_2309_09131_b200.synth import zipf_records_bucketed, zipf_tensor
    coords, vals = zipf_tensor(dims, nnz, seed=5, exponents=law)
    rec = zipf_records_bucketed(dims, nnz, seed=5, exponents=law, bucket_draws=40_000,
                                scan=100_000)
    assert rec.shape == (nnz, 4)
    np.testing.assert_array_equal(_coord_set(rec[:, :3]), _coord_set(coords))
    # values are drawn per output position
    v = rec[:, 3].view(torch.float32)
    assert torch.equal(v, vals), "values are drawn per output position"


def _both_builds(dims, law, nnz, m, g):
    from paper_2309_09131_b200 import build_device_sharded
    from paper_2309_09131_b200.layout import build_device_sharded_lean
    from paper_2309_09131_b200.synth import zipf_records_bucketed
    rec = zipf_records_bucketed(dims, nnz, seed=11, exponents=law, bucket_draws=50_000,
                                scan=1 << 18)
    k = tuple(-(-d // mm) for d, mm in zip(dims, m))
    params = params_of(dims, nnz, m, k, g, 16)
    ref = build_device_sharded(rec[:, :3].contiguous(), rec[:, 3].view(torch.float32).contiguous(),
                               params)
    lean = build_device_sharded_lean(rec.clone(), params, batch=70_000)
    return ref, lean


@pytest.mark.parametrize("dims,law,nnz,m,g", [
    ((46, 3000, 3000), (None, 1.0, 1.0), 400_000, (46, 64, 64), 2048),
    ((700, 500, 900), (1.1, 1.1, 1.1), 250_000, (16, 8, 32), 512),
])
def test_lean_build_bit_identical(dims, law, nnz, m, g):
    ref, lean = _both_builds(dims, law, nnz, m, g)
    for n in range(3):
        np.testing.assert_array_equal(lean.plan.ss_counts[n], ref.plan.ss_counts[n])
        np.testing.assert_array_equal(lean.plan.shard_offsets[n], ref.plan.shard_offsets[n])
        assert torch.equal(lean.slot_maps[n], ref.slot_maps[n]), f"slot map {n}"
    assert torch.equal(lean.crd[lean.active], ref.crd[ref.active])


def test_lean_sweep_bitwise():
    from paper_2309_09131_b200 import DeviceFactorSet, schedule_super_shards, sweep_all_modes
    dims, m = (46, 3000, 3000), (46, 64, 64)
    ref, lean = _both_builds(dims, (None, 1.0, 1.0), 400_000, m, 2048)
    fs = DeviceFactorSet.random_device(dims, 16, seed=3)
    a = sweep_all_modes(ref, fs, schedule_super_shards(ref.plan, 1))
    b = sweep_all_modes(lean, fs, schedule_super_shards(lean.plan, 1))
    for x, y in zip(a.factors, b.factors):
        assert torch.equal(x, y)
    assert torch.equal(lean.crd[lean.active], ref.crd[ref.active])
