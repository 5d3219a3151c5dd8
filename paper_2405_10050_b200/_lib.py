"""ctypes binding of the C-ABI library (include/voronray_b200.h).

This is the one place that touches the native library.  There is no CPU
fallback: importing the compute entry points without the built ``.so`` or
without a CUDA device raises :class:`~.errors.DeviceUnavailable`.
"""

from __future__ import annotations

import ctypes
import os

import torch

from ._build import LIB_PATH
from .errors import DeviceUnavailable

ABI_VERSION = 7  # vr_abi_version() of the library this package expects

_vp = ctypes.c_void_p
_i64 = ctypes.c_int64
_int = ctypes.c_int
_dbl = ctypes.c_double
_u64 = ctypes.c_uint64

# name -> argtypes (all return int status)
_SIGNATURES = {
    "vr_abi_version": [],
    "vr_record_stride": [_int],
    "vr_pack_generators": [_vp, _i64, _int, _vp, _vp, _vp],
    "vr_raycast_batch": [_vp, _i64, _int, _dbl, _vp, _vp, _vp, _i64, _vp, _vp, _vp, _int, _i64,
                         _vp, _vp, _vp, _vp, _vp, _vp, _vp],
    "vr_raycast_recheck": [_vp, _i64, _int, _vp, _vp, _i64, _vp, _vp, _vp, _int, _vp, _vp, _i64,
                           _vp, _vp, _vp, _vp, _vp],
    "vr_nearest_batch": [_vp, _i64, _int, _vp, _i64, _vp, _vp, _vp, _vp, _vp],
    "vr_verify_vertices": [_vp, _i64, _int, _vp, _vp, _i64, _dbl, _vp, _vp],
    "vr_circumcenters": [_vp, _int, _vp, _i64, _vp, _vp, _vp],
    "vr_vertex_directions": [_vp, _int, _vp, _i64, _vp, _vp, _vp],
    "vr_mc_rays": [_vp, _i64, _int, _dbl, _vp, _vp, _vp, _i64, _vp, _i64, _i64, _vp, _u64,
                   _vp, _vp, _vp, _vp, _vp, _vp],
    "vr_mc_recheck": [_vp, _i64, _int, _vp, _vp, _i64, _vp, _i64, _vp, _u64, _vp, _vp, _i64,
                      _vp, _vp, _vp, _vp],
    "vr_mc_reduce": [_vp, _int, _vp, _i64, _i64, _vp, _u64, _vp, _vp, _vp, _int, _int, _dbl,
                     _vp, _i64, _vp, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp],
    "vr_mc_directions": [_int, _i64, _vp, _i64, _u64, _vp, _vp],
    "vr_fma_probe": [_int, _int, _int, _vp, _vp],
    "vr_raycast_pruned": [_vp, _i64, _int, _dbl, _vp, _vp, _vp, _vp, _vp, _int, _i64, _vp, _vp,
                          _vp, _vp, _vp, _vp, _vp, _vp, _vp],
    "vr_mc_rays_pruned": [_vp, _i64, _int, _dbl, _vp, _vp, _vp, _i64, _i64, _vp, _u64, _vp,
                          _vp, _vp, _vp, _vp, _vp, _vp, _vp],
    "vr_pack_records32": [_vp, _i64, _int, _vp, _vp, _vp],
    "vr_pack_records32_pairs": [_vp, _i64, _int, _vp, _vp],
    "vr_pack_records_mma": [_vp, _i64, _int, _vp, _vp],
    "vr_pack_records_umma": [_vp, _i64, _int, _vp, _vp],
    "vr_host_streams": [ctypes.c_uint64, ctypes.c_uint64, _vp, _i64, _vp],
    "vr_descent_directions": [_vp, _int, _vp, _vp, _vp, _i64, ctypes.c_double, _vp, _vp, _vp,
                              _vp],
    "vr_trav_level_open": [_vp, _int, _vp, _i64, _vp, _vp, _vp, _vp, _vp, _i64, _vp],
    "vr_trav_level_cast": [_vp, _vp, _i64, _int, ctypes.c_double, _vp, _vp, _vp, _vp, _i64,
                           _vp, _vp, _i64, ctypes.c_int32, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                           _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _vp],
    "vr_host_normals": [_vp, _vp, _i64, _i64, _vp],
    "vr_ray_keys": [_vp, _vp, _int, _i64, _vp, _i64, _int, _vp, _vp],
    "vr_ray_order": [_vp, _vp, _int, _i64, _vp, _i64, _int, _i64, _vp, _vp, _vp, _vp],
    "vr_screen32_stats": [_vp, _i64, _int, _vp, _vp, _vp],
    "vr_prune_index_layout": [_i64, _int, _int, _vp],
    "vr_build_prune_index": [_vp, _i64, _int, _vp, _int, _vp, _i64, _vp, _i64, _vp, _vp],
    "vr_trav_level_workspace": [_i64, _i64, _i64, _int, _vp],
    "vr_trav_run_workspace": [_i64, _i64, _i64, _int, _vp],
    "vr_trav_run": [_vp, _vp, _vp, _i64, _int, _dbl, _vp, _vp, ctypes.c_int32, _vp, _i64, _vp,
                    _vp, _i64, _vp],
    "vr_shard_bucket": [_vp, _i64, _int, _int, _vp, _vp, _vp, _vp, _vp],
    "vr_shard_gather_rows": [_vp, _int, _vp, _i64, _vp, _vp],
    "vr_shard_scatter_rows": [_vp, _int, _vp, _i64, _vp, _vp],
    "vr_shard_open": [_vp, _i64, _int, _vp, _vp, _vp, _vp, _vp, _vp, _vp],
    "vr_trav_claim_sigma": [_vp, _int, _vp, _i64, ctypes.c_int32, _vp, _vp, _vp],
    "vr_trav_bump_keys": [_vp, _int, _vp, _i64, _vp, _vp],
    "vr_vertex_edges": [_vp, _i64, _int, _vp, _vp],
    "vr_trav_level_rays": [_vp, _i64, _int, _dbl, _vp, _vp, _vp, _vp, _i64, _vp, _vp, _i64, _vp,
                           _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _vp],
    "vr_lex_order": [_vp, _i64, _int, _vp, _vp, _vp, _vp],
    "vr_edge_incidence": [_vp, _i64, _int, _vp, _vp, _vp, _vp, _vp, _vp],
    "vr_edge_check": [_vp, _vp, _i64, _vp, _i64, _int, _vp, _vp],
    "vr_hmc_face_index": [_vp, _i64, _int, _i64, _vp, _vp, _i64, _vp, _vp, _vp, _vp, _vp, _vp,
                          _vp, _vp, _vp],
    "vr_hmc_faces": [_vp, _vp, _i64, _vp, _i64, _vp, _int, _vp, _vp, _vp, _i64, _int, _vp, _vp,
                     _vp, _vp, _vp, _vp, _vp, _vp],
    "vr_hmc_cells": [_vp, _int, _vp, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _int, _vp, _vp,
                     _vp, _vp, _vp, _vp],
    "vr_mc_integrate": [_vp, _int, _vp, _i64, _i64, _vp, _u64, _vp, _vp, _vp, _int, _dbl, _int,
                        _vp, _int, _vp, _vp, _i64, _vp, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                        _vp, _vp],
    "vr_mc_uniforms": [_i64, _vp, _i64, _int, _u64, _vp, _vp],
    "vr_record32_stride": [_int],
    "vr_trav_insert_vertices": [_vp, _int, _vp, _i64, ctypes.c_int32, ctypes.c_int32, _int, _vp],
    "vr_trav_rehash_edges": [_vp, _int, _vp, _vp, _vp, _i64, _vp],
    "vr_trav_open_edges": [_vp, _int, _vp, _i64, _vp, _vp, _vp],
    "vr_trav_open_edges_sub": [_vp, _int, _vp, _i64, _int, _int, _vp, _vp, _vp],
    "vr_trav_set_sub_rounds": [_i64, _int],
    "vr_trav_emit_rays": [_vp, _int, _vp, _vp, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp],
    "vr_trav_claim": [_vp, _int, _vp, _vp, _vp, _i64, ctypes.c_int32, _vp, _vp, _vp, _vp, _vp],
    "vr_trav_finalize": [_vp, _vp, _int, _vp, _vp, _vp, _vp, _i64, ctypes.c_int32, _vp, _vp,
                         _vp, _int, _vp],
    "vr_trav_boundary": [_int, _vp, _vp, _vp, _vp, _i64, _vp, _i64, _vp, _vp, _vp],
    "vr_trav_published": [_vp, _i64, _vp, _vp],
    "vr_trav_edge_compact": [_vp, _int, _vp, _vp, _vp, _vp],
    "vr_trav_edges_count": [_vp, _vp, _vp, _vp, _vp, _vp],
    "vr_trav_edges_compact": [_vp, _int, _vp, _i64, _vp, _vp, _vp, _vp],
}

# Symbols declared in include/voronray_b200.h that the .so must export.
EXPORTED = tuple(_SIGNATURES) + ("vr_status_string", "vr_record_rows", "vr_mc_map_bytes")

_LIB = None


def load_library():
    """Load the shared library (no device needed); raises if it was not built."""
    global _LIB
    if _LIB is not None:
        return _LIB
    path = os.environ.get("VR_LIB_PATH", LIB_PATH)  # debug builds (tools/stats_build.sh)
    if not os.path.exists(path):
        raise DeviceUnavailable(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
            "g.build()'` (nvcc, sm_100a). There is no CPU fallback.")
    lib = ctypes.CDLL(path)
    for name, argtypes in _SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = argtypes
        fn.restype = ctypes.c_int
    lib.vr_mc_map_bytes.argtypes = [_i64, _int, _int]
    lib.vr_mc_map_bytes.restype = ctypes.c_int64
    lib.vr_record_rows.argtypes = [_i64]
    lib.vr_record_rows.restype = ctypes.c_int64
    lib.vr_status_string.argtypes = [_int]
    lib.vr_status_string.restype = ctypes.c_char_p
    _LIB = lib
    return lib


_HAVE_DEVICE = False


def lib():
    """The library, after checking that a CUDA device is present (checked
    until it succeeds once: torch.cuda.is_available() costs ~10 us per call,
    and the traversal calls this hundreds of times per diagram)."""
    global _HAVE_DEVICE
    L = load_library()
    if not _HAVE_DEVICE:
        if not torch.cuda.is_available():
            raise DeviceUnavailable("no CUDA device: the B200 kernels have no CPU fallback")
        _HAVE_DEVICE = True
    return L


REC_PAD = 512


def record_rows(n):
    """Rows of a padded record array (include/voronray_b200.h vr_record_rows)."""
    return (int(n) + REC_PAD - 1) // REC_PAD * REC_PAD


def check(status, what=""):
    if status != 0:
        msg = load_library().vr_status_string(int(status)).decode()
        raise RuntimeError(f"{what or 'voronray_b200'} failed: {msg} (status {status})")


def ptr(t):
    """Raw device pointer of a tensor (or None)."""
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def stream_handle(stream=None):
    """cudaStream_t of `stream`, or of torch's current stream on the current
    device (raw C binding: torch.cuda.current_stream() costs ~15 us)."""
    if stream is not None:
        return ctypes.c_void_p(stream.cuda_stream)
    return ctypes.c_void_p(torch._C._cuda_getCurrentRawStream(torch._C._cuda_getDevice()))


def to_host(t):
    """Device tensor -> numpy through a pinned staging buffer (pageable
    .cpu() copies of large arrays run several times slower)."""
    import torch
    t = t.contiguous()
    if t.is_cuda and t.numel() > (1 << 16):
        buf = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
        buf.copy_(t)
        return buf.numpy()
    return t.cpu().numpy()

