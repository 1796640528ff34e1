"""FLYCOO image and MCFD dumps with device tensors."""
import numpy as np
import pytest
import torch

from gpu_helpers import factors_f32, host_records
from paper_2309_09131_b200 import (DeviceFactorSet, build_device_sharded, device_params,
                                   mttkrp_mode, schedule_super_shards, sweep_all_modes)
from paper_2309_09131_b200 import io as fio
from paper_2309_09131_b200.synth import zipf_tensor

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dims", [(3000, 2000, 2500), (300, 400, 250, 90)])
def test_flycoo_image_roundtrip(tmp_path, dims):
    coords, vals = zipf_tensor(dims, 300_000, seed=4, exponents=(1.1,) * len(dims))
    params = device_params(dims, 300_000, 32, g=4096)
    st = build_device_sharded(coords, vals, params)
    fs = DeviceFactorSet.random_device(dims, 32, seed=1)
    smap = schedule_super_shards(st.plan, 1)
    mttkrp_mode(st, fs, 0, smap)  # save a non-zero active mode
    path = tmp_path / "t.flycoo"
    fio.save_flycoo(st, path)
    st2 = fio.load_flycoo(path)
    assert st2.active_mode == st.active_mode
    for key in ("ss_counts", "shard_offsets", "ss_first_shard"):
        for a, b in zip(getattr(st.plan, key), getattr(st2.plan, key)):
            assert np.array_equal(a, b)
    assert np.array_equal(host_records(st)[0], host_records(st2)[0])
    assert np.array_equal(host_records(st)[1], host_records(st2)[1])
    for a, b in zip(st.slot_maps, st2.slot_maps):
        assert torch.equal(a, b)
    n = st.active_mode
    assert torch.equal(mttkrp_mode(st, fs, n, smap), mttkrp_mode(st2, fs, n, smap))


def test_mcfd_roundtrip_device(tmp_path):
    fs = DeviceFactorSet.random_device((50, 70, 30), 8, seed=3)
    fs.lambdas[:] = [1, 2, 3, 4, 5, 6, 7, 8]
    p = tmp_path / "f.mcfd"
    fio.save_factor_set(fs, p)
    back = fio.load_factor_set(p)
    assert all(torch.equal(a, b) for a, b in zip(fs.factors, back.factors))
    assert np.array_equal(back.lambdas, fs.lambdas)
