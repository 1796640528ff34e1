"""The reference-side binding a maintainer would add next to modecycle's
``_kernels.py`` to keep the reference engine and swap only its kernel
(INTEGRATION.md section 2): ctypes over the C ABI of include/flycoo.h.
Exercised by tests/test_gpu_binding.py (GPU) and tests/test_abi.py (CPU:
argument list against the header)."""
import ctypes
from pathlib import Path

import torch

LIB_PATH = Path(__file__).resolve().parents[1] / "paper_2309_09131_b200" / "libflycoo.so"
vp, i64, c_int = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
MODE_WORKER_ARGTYPES = [vp, vp, vp, vp, vp, vp, vp, c_int, c_int, c_int, i64, i64,
                        vp, vp, vp, vp, i64, i64, i64, vp, i64, vp, i64, vp, vp,
                        vp, i64, c_int, c_int, c_int, vp, vp, vp]
_lib = None


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(str(LIB_PATH))
        L.fc_mode_worker.restype = c_int
        L.fc_mode_worker.argtypes = MODE_WORKER_ARGTYPES
        L.fc_last_error.restype = ctypes.c_char_p
        _lib = L
    return _lib


def mode_worker_b200(src_crd, src_val, dst_crd, dst_val, factors, out, mode, plan, work,
                     slots, flags, counters, do_compute=True, do_remap=True):
    """Replaces _kernels.mode_worker (_kernels.py:38-88) + the thread fan-out of
    engine.mttkrp_mode (engine.py:229-245): one stream-ordered call per mode."""
    L = lib()
    fptrs = (ctypes.c_void_p * len(factors))(*[f.data_ptr() for f in factors])
    rc = L.fc_mode_worker(
        src_crd.data_ptr(), src_val.data_ptr() if src_val is not None else None,
        dst_crd.data_ptr(), dst_val.data_ptr() if dst_val is not None else None,
        fptrs, (ctypes.c_int64 * len(factors))(*plan.params.dims), out.data_ptr(),
        len(factors), mode, out.shape[1], out.shape[0], plan.params.m[mode],
        work.chunk_start.data_ptr(), work.chunk_ss.data_ptr(), work.chunk_part.data_ptr(),
        work.chunk_rows.data_ptr() if work.chunk_rows is not None else None,
        work.tile_rows, work.hist_rows, work.nchunks,
        work.red1.data_ptr(), work.nred1, work.red2.data_ptr(), work.nred2,
        work.part_ws.data_ptr() if work.part_ws is not None else None,
        work.part_ws2.data_ptr() if work.part_ws2 is not None else None,
        slots.data_ptr(), src_crd.shape[0], int(do_compute), int(do_remap),
        int(work.acc_in_smem), flags.data_ptr(), counters.data_ptr(),
        torch.cuda.current_stream().cuda_stream)
    if rc != 0:
        raise RuntimeError(L.fc_last_error().decode())
