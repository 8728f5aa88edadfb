"""ctypes bindings of the test-only checkers (see oracle/oracle.c header).

TEST INFRASTRUCTURE ONLY -- imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs, never by the product package.

* ``orc()``  -> liboracle.so: CPU restatement of the kernels ("parity unpinned"
  by the reference for kernel *results*: the reference has no executing
  kernel; cross-checked against numpy/scipy in tests/).
* ``ref()``  -> _ref/librooflens_ref.so: the reference library itself (built
  from /root/reference/proj/src by oracle/Makefile) behind an extern "C" shim;
  pins the accounting (W/Q), bounds and spec parsing.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "librooflens_ref.so")

_u64, _i64, _dbl, _int, _ptr = C.c_uint64, C.c_int64, C.c_double, C.c_int, C.c_void_p
_U64P, _DP = C.POINTER(_u64), C.POINTER(_dbl)

_ORC_SIGS = {
    "orc_mix": (_u64, [_u64, _u64]),
    "orc_key": (_u64, [_u64, _u64]),
    "orc_fill_uniform": (None, [_ptr, _u64, _u64, _u64, _u64, _int]),
    "orc_scale": (None, [_ptr, _ptr, _dbl, _u64]),
    "orc_gen_band_csr": (_int, [_u64, _u64, _u64, C.c_uint32, _u64, _u64, _ptr, _ptr, _ptr]),
    "orc_gemv": (None, [_u64, _u64, _ptr, _ptr, _ptr]),
    "orc_spmv_csr": (None, [_u64, _ptr, _ptr, _ptr, _ptr, _i64, _ptr]),
    "orc_preset_points": (_int, [C.c_char_p]),
    "orc_preset_offsets": (_int, [C.c_char_p, _ptr]),
    "orc_default_weights": (_int, [C.c_char_p, _ptr]),
    "orc_stencil_init": (None, [_ptr, _u64, _u64, _u64, _int, _u64, _u64, _int, _u64]),
    "orc_stencil": (_int, [C.c_char_p, _U64P, _ptr, _u64, _ptr, _ptr]),
    "orc_stencil_sweep": (_int, [C.c_char_p, _U64P, _ptr, _u64, _u64, _ptr, _ptr]),
    "orc_rel_err": (_dbl, [_ptr, _ptr, _u64]),
    "orc_bit_mismatches": (_u64, [_ptr, _ptr, _u64]),
    "orc_num_threads": (_int, []),
}

_REF_SIGS = {
    "ref_last_error": (C.c_char_p, []),
    "ref_scale_model": (_int, [_u64, _int, _U64P, _U64P]),
    "ref_gemv_model": (_int, [_u64, _u64, _int, _U64P, _U64P]),
    "ref_spmv_generic_model": (_int, [_u64, _u64, _u64, _u64, _u64, _u64, _u64, _int, _U64P, _U64P]),
    "ref_spmv_csr_model": (_int, [_u64, _u64, _u64, _u64, _int, _U64P, _U64P]),
    "ref_stencil_model": (_int, [C.c_char_p, _int, _u64, _U64P, _U64P, _U64P]),
    "ref_intensity_ratio": (_int, [_u64, _u64, _U64P, _U64P]),
    "ref_load_spec": (_int, [C.c_char_p, _DP, _DP, _DP, _DP]),
    "ref_builtin_spec": (_int, [C.c_char_p, _DP, _DP, _DP, _DP]),
    "ref_machine_balance": (_int, [_dbl, _dbl, _dbl, _int, _DP]),
    "ref_tensor_alpha": (_int, [_dbl, _dbl, _dbl, _DP]),
    "ref_attainable": (_int, [_dbl, _dbl, _dbl, _int, _dbl, _DP]),
    "ref_classify": (_int, [_dbl, _dbl]),
    "ref_spec_eval": (_int, [C.c_char_p, _int, _int, _int, _dbl, _DP]),
    "ref_serialize_spec": (_int, [C.c_char_p, C.c_char_p, _u64]),
    "ref_load_spec_file": (_int, [C.c_char_p, _DP]),
    "ref_mem_cmp_ratio": (_int, [_dbl, _dbl, _DP]),
    "ref_overlapped_total": (_int, [_dbl, _dbl, _dbl, _DP]),
    "ref_sample_curve": (_int, [_dbl, _dbl, _dbl, _int, _dbl, _dbl, _u64, _ptr, _ptr, _u64, _U64P]),
    "ref_kernel_speedup_ceiling": (_int, [_dbl, _dbl, _dbl, _DP, C.POINTER(_int)]),
    "ref_bound_text": (_int, [_int, _dbl, _dbl, _dbl, _dbl, _DP, C.POINTER(_int), C.POINTER(_int),
                              C.POINTER(_int), C.c_char_p, C.c_uint64, C.c_char_p, C.c_uint64]),
    "ref_tensor_core_ceiling": (_int, [_dbl, _DP]),
    "ref_workload_ceiling": (_int, [_dbl, _dbl, _DP]),
    "ref_unoverlapped_speedup": (_int, [_dbl, _dbl, _dbl, _dbl, _DP]),
    "ref_min_temporal_depth": (_int, [_dbl, _dbl, _U64P]),
    "ref_tc_scale_trick_throughput": (_int, [_dbl, _u64, _u64, _DP]),
    "ref_parse_stats_file": (_int, [C.c_char_p, _U64P, _U64P, _U64P]),
    "ref_stats_to_report": (_int, [_u64, _u64, _u64, _dbl, _dbl, _dbl, _dbl, _U64P, _U64P, C.POINTER(_int), _DP,
                                   C.POINTER(_int), _DP, _U64P, C.POINTER(_int)]),
}

_orc = None
_ref = None


def _load(path, sigs):
    L = C.CDLL(path)
    for name, (res, args) in sigs.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    return L


def orc():
    global _orc
    if _orc is None:
        _orc = _load(ORACLE_SO, _ORC_SIGS)
    return _orc


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref():
    global _ref
    if _ref is None:
        _ref = _load(REF_SO, _REF_SIGS)
    return _ref


def _p(a: np.ndarray) -> int:
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data


# --- convenience wrappers over numpy arrays ---------------------------------
def fill_uniform(n, seed, stream_id, idx0=0, kind=0) -> np.ndarray:
    out = np.empty(n, np.float64)
    orc().orc_fill_uniform(_p(out), n, seed, stream_id, idx0, kind)
    return out


def scale(b: np.ndarray, q: float) -> np.ndarray:
    a = np.empty_like(b)
    orc().orc_scale(_p(a), _p(b), q, b.size)
    return a


def gen_band_csr(m_local, row0, n, k, hb, seed):
    rp = np.empty(m_local + 1, np.int32)
    col = np.empty(m_local * k, np.int32)
    val = np.empty(m_local * k, np.float64)
    rc = orc().orc_gen_band_csr(m_local, row0, n, k, hb, seed, _p(rp), _p(col), _p(val))
    if rc:
        raise ValueError("orc_gen_band_csr: bad arguments")
    return rp, col, val


def spmv_csr(rp, col, val, x, col_base=0) -> np.ndarray:
    m = rp.size - 1
    y = np.empty(m, np.float64)
    orc().orc_spmv_csr(m, _p(rp), _p(col) if col.size else None, _p(val) if val.size else None,
                       _p(x) if x.size else None, col_base, _p(y))
    return y


def gemv(A: np.ndarray, x: np.ndarray) -> np.ndarray:
    A = np.ascontiguousarray(A, np.float64)
    y = np.empty(A.shape[0], np.float64)
    orc().orc_gemv(A.shape[0], A.shape[1], _p(A), _p(np.ascontiguousarray(x, np.float64)), _p(y))
    return y


def default_weights(preset: str) -> np.ndarray:
    w = np.empty(64, np.float64)
    n = orc().orc_default_weights(preset.encode(), _p(w))
    return w[:n].copy()


def stencil_init(shape, radius, seed, outer_begin=0, outer_end=None, global_shape=None):
    """Field of `shape` (ny, nx) or (nz, ny, nx); with global_shape it is the
    slab of outer indices [outer_begin, outer_end) of that global grid."""
    gs = tuple(global_shape or shape)
    if outer_end is None:
        outer_end = outer_begin + shape[0]
    u = np.empty(shape, np.float64)
    if len(gs) == 2:
        orc().orc_stencil_init(_p(u), gs[1], gs[0], 1, 2, outer_begin, outer_end, radius, seed)
    else:
        orc().orc_stencil_init(_p(u), gs[2], gs[1], gs[0], 3, outer_begin, outer_end, radius, seed)
    return u


def stencil(preset: str, u: np.ndarray, steps: int, weights=None) -> np.ndarray:
    """Runs `steps` sweeps on copies; returns the final field."""
    a = np.ascontiguousarray(u).copy()
    b = a.copy()
    if a.ndim == 2:
        dims = (_u64 * 3)(a.shape[1], a.shape[0], 1)
    else:
        dims = (_u64 * 3)(a.shape[2], a.shape[1], a.shape[0])
    w = None
    if weights is not None:
        w = np.ascontiguousarray(weights, np.float64)
    rc = orc().orc_stencil(preset.encode(), dims, _p(w) if w is not None else None, steps,
                           _p(a), _p(b))
    if rc:
        raise ValueError(f"orc_stencil rc={rc}")
    return a if steps % 2 == 0 else b


def stencil_sweep(preset: str, u: np.ndarray, v: np.ndarray, o0: int, o1: int, weights=None) -> None:
    """v = S(u) over outer indices [o0, o1) of u's own grid (in place into v)."""
    assert u.flags["C_CONTIGUOUS"] and v.flags["C_CONTIGUOUS"] and u.shape == v.shape
    if u.ndim == 2:
        dims = (_u64 * 3)(u.shape[1], u.shape[0], 1)
    else:
        dims = (_u64 * 3)(u.shape[2], u.shape[1], u.shape[0])
    w = None if weights is None else np.ascontiguousarray(weights, np.float64)
    rc = orc().orc_stencil_sweep(preset.encode(), dims, _p(w) if w is not None else None, o0, o1,
                                 _p(u), _p(v))
    if rc:
        raise ValueError(f"orc_stencil_sweep rc={rc}")


def rel_err(a: np.ndarray, b: np.ndarray) -> float:
    a = np.ascontiguousarray(a, np.float64).ravel()
    b = np.ascontiguousarray(b, np.float64).ravel()
    return float(orc().orc_rel_err(_p(a), _p(b), a.size))


def bit_mismatches(a: np.ndarray, b: np.ndarray) -> int:
    a = np.ascontiguousarray(a, np.float64).ravel()
    b = np.ascontiguousarray(b, np.float64).ravel()
    return int(orc().orc_bit_mismatches(_p(a), _p(b), a.size))


def num_threads() -> int:
    return int(orc().orc_num_threads())
