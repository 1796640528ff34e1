"""ctypes binding of libflycoo.so (include/flycoo.h).

There is no CPU fallback: if the library is missing or no CUDA device is
present, every entry point raises.  Build it with ``__graft_entry__.build()``
(or ``make -C paper_2309_09131_b200/csrc``).
"""

from __future__ import annotations

import ctypes
import threading
from pathlib import Path

import os

_HERE = Path(__file__).resolve().parent
# FLYCOO_LIB selects an alternative in-tree build (A/B kernel experiments)
LIB_PATH = _HERE / os.environ.get("FLYCOO_LIB", "libflycoo.so")

_c = ctypes
_vp = _c.c_void_p
_i64 = _c.c_int64
_int = _c.c_int

# name -> (restype, argtypes); every pointer is passed as void* (device or
# host address as an int), sizes as int64.
_SIGS = {
    "fc_version": (_int, []),
    "fc_last_error": (_c.c_char_p, []),
    "fc_crd_words": (_int, [_int]),
    "fc_value_embedded": (_int, [_int]),
    "fc_smem_acc_rows_max": (_i64, [_int]),
    "fc_tile_elems": (_int, []),
    "fc_set_kernel_variant": (_int, [_int, _int]),
    "fc_chunk_rows_max": (_i64, [_int, _int, _i64]),
    "fc_mode_worker": (_int, [
        _vp, _vp, _vp, _vp,            # src_crd, src_val, dst_crd, dst_val
        _vp, _vp, _vp,                 # factors (host array of device ptrs), dims (host), out
        _int, _int, _int,              # nmodes, mode, rank
        _i64, _i64,                    # out_rows, m_mode
        _vp, _vp, _vp, _vp, _i64, _i64, _i64,  # chunk_start/ss/part/rows, tile_rows, hist_rows, nchunks
        _vp, _i64, _vp, _i64,          # red1, nred1, red2, nred2
        _vp, _vp, _vp, _i64,           # part_ws, part_ws2, dest_slots, nnz
        _int, _int, _int,              # do_compute, do_remap, acc_in_smem
        _vp, _vp, _vp]),               # flags, counters, stream
    "fc_mode_worker_peers": (_int, [
        _vp, _vp,                      # src_crd, src_val
        _vp, _vp, _vp,                 # factors (host array of device ptrs), dims (host), out
        _int, _int, _int,              # nmodes, mode, rank
        _i64, _i64,                    # out_rows, m_mode
        _vp, _vp, _vp, _vp, _i64, _i64, _i64,  # chunk_start/ss/part/rows, tile_rows, hist_rows, nchunks
        _vp, _i64, _vp, _i64,          # red1, nred1, red2, nred2
        _vp, _vp, _vp, _i64,           # part_ws, part_ws2, dest_slots (global), nnz (local)
        _int, _int,                    # do_compute, acc_in_smem
        _vp, _vp,                      # flags, counters
        _int, _vp, _vp, _vp,           # npeers, peer_crd, peer_val (host arrays), peer_base (host)
        _vp, _vp,                      # peer_part_ws (host array), chunk_owner (device int32)
        _vp]),
    "fc_mode_worker_peers_planned": (_int, [
        _vp, _vp,                      # src_crd, src_val
        _vp, _vp, _vp,                 # factors (host array of device ptrs), dims (host), out
        _int, _int, _int,              # nmodes, mode, rank
        _i64, _i64,                    # out_rows, m_mode
        _vp, _vp, _vp, _vp, _i64, _i64, _i64,  # chunk_start/ss/part/rows, tile_rows, hist_rows, nchunks
        _vp, _i64, _vp, _i64,          # red1, nred1, red2, nred2
        _vp, _vp, _vp, _i64,           # part_ws, part_ws2, dest_slots (global), nnz (local)
        _int, _int,                    # do_compute, acc_in_smem
        _vp, _vp,                      # flags, counters
        _int, _vp, _vp, _vp,           # npeers, peer_crd, peer_val (host arrays), peer_base (host)
        _vp, _vp,                      # peer_part_ws (host array), chunk_owner (device int32)
        _vp, _vp,                      # tile_perm, tile_bins (device uint16, or NULL)
        _vp]),                         # stream
    "fc_reduce_partials": (_int, [_vp, _i64, _vp, _i64, _vp, _vp, _vp, _i64, _i64, _int, _vp]),
    "fc_tile_plan_emit": (_int, [
        _vp, _vp, _vp, _vp,            # src_crd, src_val, factors, dims
        _int, _int, _int, _i64, _i64,  # nmodes, mode, rank, out_rows, m_mode
        _vp, _vp, _vp, _vp, _i64, _i64, _i64,  # chunk_start/ss/part/rows, tile_rows, hist_rows, nchunks
        _i64, _vp, _vp,                # nnz, flags, counters
        _vp, _vp, _vp]),               # tile_perm, tile_bins, stream
    "fc_tile_plan_keys": (_i64, [_i64, _i64]),
    "fc_mode_worker_planned": (_int, [
        _vp, _vp, _vp, _vp,            # src_crd, src_val, dst_crd, dst_val
        _vp, _vp, _vp,                 # factors, dims, out
        _int, _int, _int,              # nmodes, mode, rank
        _i64, _i64,                    # out_rows, m_mode
        _vp, _vp, _vp, _vp, _i64, _i64, _i64,  # chunk_start/ss/part/rows, tile_rows, hist_rows, nchunks
        _vp, _i64, _vp, _i64,          # red1, nred1, red2, nred2
        _vp, _vp, _vp, _i64,           # part_ws, part_ws2, dest_slots, nnz
        _int, _vp, _vp,                # do_remap, flags, counters
        _vp, _vp, _vp]),               # tile_perm, tile_bins, stream
    "fc_ipc_handle_bytes": (_int, []),
    "fc_ipc_alloc": (_int, [_i64, _vp]),
    "fc_ipc_free": (_int, [_vp]),
    "fc_ipc_handle": (_int, [_vp, _vp]),
    "fc_ipc_open": (_int, [_vp, _vp]),
    "fc_ipc_close": (_int, [_vp]),
    "fc_copy_async": (_int, [_vp, _vp, _i64, _vp]),
    "fc_gather_peer_rows": (_int, [_vp, _vp, _vp, _int, _int, _i64, _vp]),
    "fc_stream_signal": (_int, [_vp, _c.c_uint32, _vp]),
    "fc_stream_wait": (_int, [_vp, _c.c_uint32, _vp]),
    "fc_stream_wait_flush_supported": (_int, []),
    "fc_remap_cursor": (_int, [_vp, _vp, _vp, _vp, _vp, _vp, _int, _int, _i64, _vp, _vp, _vp, _vp]),
    "fc_scatter_records": (_int, [_vp, _vp, _i64, _vp, _vp, _i64, _vp, _int, _vp, _vp, _vp]),
    "fc_build_morton": (_int, [_vp, _i64, _int, _vp, _vp, _vp, _vp, _vp]),
    "fc_build_sort_temp_bytes": (_i64, [_i64]),
    "fc_build_sort_pairs": (_int, [_vp, _vp, _vp, _vp, _i64, _int, _vp, _i64, _vp]),
    "fc_build_gather_key": (_int, [_vp, _i64, _int, _vp, _vp, _vp, _int, _int, _i64, _int, _vp, _vp]),
    "fc_build_ss_hist": (_int, [_vp, _i64, _int, _int, _i64, _i64, _vp, _vp]),
    "fc_build_shard_ids": (_int, [_vp, _i64, _vp, _int, _int, _i64, _vp, _vp, _i64, _vp, _vp]),
    "fc_build_device_key": (_int, [_vp, _i64, _vp, _vp, _vp, _vp]),
    "fc_build_invert": (_int, [_vp, _i64, _vp, _vp]),
    "fc_build_slots": (_int, [_vp, _vp, _i64, _vp, _vp]),
    "fc_build_records": (_int, [_vp, _i64, _int, _vp, _vp, _vp, _vp, _vp]),
    "fc_build_slots_scatter": (_int, [_vp, _vp, _i64, _vp, _vp]),
    "fc_build_records_scatter": (_int, [_vp, _i64, _int, _vp, _vp, _vp, _vp, _vp]),
    "fc_build_iota": (_int, [_vp, _i64, _vp]),
    "fc_build_morton32": (_int, [_vp, _i64, _int, _int, _vp, _vp, _vp, _vp]),
    "fc_build_sort32_temp_bytes": (_i64, [_i64]),
    "fc_build_sort_pairs32": (_int, [_vp, _vp, _vp, _vp, _i64, _int, _vp, _i64, _vp]),
    "fc_build_iv_key32": (_int, [_vp, _i64, _vp, _int, _int, _i64, _vp, _vp]),
    "fc_build_gather_u32": (_int, [_vp, _i64, _vp, _vp, _vp]),
    "fc_build_scatter_rec16": (_int, [_vp, _i64, _vp, _vp, _vp]),
    "fc_synth_draw_at": (_int, [_c.c_uint64, _vp, _i64, _int, _vp, _vp, _vp, _int, _int, _vp, _int, _vp]),
    "fc_synth_draw": (_int, [_c.c_uint64, _i64, _int, _vp, _vp, _vp, _vp, _vp]),
    "fc_synth_keys": (_int, [_vp, _i64, _int, _vp, _vp, _vp, _vp]),
    "fc_synth_mark_first": (_int, [_vp, _vp, _vp, _i64, _vp, _vp]),
    "fc_synth_uniform": (_int, [_c.c_uint64, _c.c_uint32, _i64, _vp, _int, _vp]),
}

ERR_UNSUPPORTED = -2  # FC_ERR_UNSUPPORTED (flycoo.h)

_lib = None
_lock = threading.Lock()


class FlycooError(RuntimeError):
    """A libflycoo entry point returned an error code."""


def load():
    """Load libflycoo.so (raises if it was not built)."""
    global _lib
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise RuntimeError(
                    f"{LIB_PATH} is missing: the CUDA extension was not built "
                    "(run __graft_entry__.build()); there is no CPU fallback")
            L = ctypes.CDLL(str(LIB_PATH))
            for name, (res, args) in _SIGS.items():
                f = getattr(L, name)
                f.restype = res
                f.argtypes = args
            _lib = L
    return _lib


def exported_symbols() -> list[str]:
    return list(_SIGS)


def call(name: str, *args) -> int:
    """Call an int-returning entry point; raise FlycooError on failure."""
    L = load()
    rc = getattr(L, name)(*args)
    if rc != 0:
        msg = L.fc_last_error().decode(errors="replace")
        raise FlycooError(f"{name} failed ({rc}): {msg}")
    return rc


def ptr_array(ptrs) -> ctypes.Array:
    """Host array of device pointers (const float *const *)."""
    arr = (ctypes.c_void_p * len(ptrs))(*[p if p else None for p in ptrs])
    return arr


def i64_array(vals) -> ctypes.Array:
    return (ctypes.c_int64 * len(vals))(*[int(v) for v in vals])
