"""GPU: INTEGRATION.md section 2's reference-side ctypes binding
(tests/reference_binding.py, the module a maintainer would add next to the
reference's _kernels.py) drives one mode pass through the C ABI directly;
its output matches the oracle and its remapped buffer equals the package
engine's, bit-exactly."""
import numpy as np
import pytest
import torch

import oracle
import reference_binding as rb
from gpu_helpers import assert_rel, factors_f32, host_records
from paper_2309_09131_b200 import (DeviceFactorSet, build_device_sharded, device_params,
                                   mttkrp_mode, schedule_super_shards)
from paper_2309_09131_b200.synth import synth_tensor

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("mode_m", [(0, 32), (1, 600)])  # shared-memory tile / global accumulator
def test_reference_binding_mode_pass(mode_m):
    mode, m = mode_m
    dims = (400, 350, 300)
    subs, vals = synth_tensor(dims, 100_000, seed=4, skew=0.6)
    vals = vals.astype(np.float32).astype(np.float64)
    params = device_params(dims, len(vals), 32, g=4096, m=[m] * 3)
    fs = factors_f32(dims, 32, 8)
    st = build_device_sharded(subs, vals, params)
    ref = build_device_sharded(subs, vals, params)
    smap = schedule_super_shards(ref.plan, 1)
    dfs = DeviceFactorSet.from_host(fs)
    for n in range(mode):  # bring both tensors to `mode` through the engine
        mttkrp_mode(st, dfs, n, smap)
        mttkrp_mode(ref, dfs, n, smap)
    work = st.mode_work(mode, 32)
    out = torch.zeros((dims[mode], 32), dtype=torch.float32, device="cuda")
    flags = torch.zeros(1, dtype=torch.int32, device="cuda")
    counters = torch.zeros(1, dtype=torch.int64, device="cuda")
    a, b = st.active, 1 - st.active
    rb.mode_worker_b200(st.crd[a], st.val[a], st.crd[b], st.val[b], list(dfs.factors), out, mode,
                        st.plan, work, st.slot_maps[mode], flags, counters)
    torch.cuda.synchronize()
    assert int(flags.item()) == 0 and int(counters.item()) == st.nnz
    want = oracle.reference_mttkrp(subs, vals, [f.astype(np.float64) for f in fs], mode)
    assert_rel(out.double().cpu().numpy(), want, what=f"binding mode {mode}")
    got_eng = mttkrp_mode(ref, dfs, mode, smap)
    assert torch.equal(out, got_eng)
    assert torch.equal(st.crd[b], ref.crd[ref.active])
