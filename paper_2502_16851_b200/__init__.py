"""B200-native (sm_100a) FP64 memory-bound kernels of arXiv 2502.16851.

Python host side of the framework: a thin ctypes binding of the C-ABI in
``include/rooflens_b200.h`` (the library ``librooflens_b200.so`` built in-tree
from ``csrc/``), mirroring the reference's kernel identities
(``/root/reference/proj/include/rooflens/kernels.hpp:84-105``):

* accounting -- ``scale_model``, ``gemv_model``, ``spmv_generic_model``,
  ``spmv_csr_model``, ``stencil_model``, ``stencil_preset`` (pure host);
* executing kernels -- ``scale``, ``spmv_csr``, ``stencil`` (+ ``*_rows`` /
  ``*_sweep`` partial forms and ``*_host`` end-to-end forms), each with a
  CUDA-core and a tensor-core variant selected by ``unit``;
* hardware spec / roofline / bounds -- ``load_spec``, ``builtin_spec``,
  ``machine_balance``, ``tensor_alpha``, ``attainable``, ``classify``,
  ``kernel_speedup_ceiling``, ``tensor_core_ceiling``, ``workload_ceiling``,
  ``min_temporal_depth``, ``tc_scale_trick_throughput``.

Errors mirror the reference's ``rooflens::Error`` (error.hpp:36-46): a
``RooflensError`` whose ``kind`` is the ErrorKind name and whose message is
``"<Kind>: <msg>"``.  There is no CPU fallback: every executing call runs the
sm_100a kernels or raises.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import Optional, Sequence

__all__ = [
    "CUDA_CORE", "TENSOR_CORE", "FP64", "FP32", "FP16", "RooflensError", "KernelCharacterization",
    "HardwareSpec", "lib", "library_path", "scale_model", "gemv_model", "spmv_generic_model",
    "spmv_csr_model", "stencil_model", "stencil_preset", "stencil_default_weights", "scale",
    "gemv", "spmv_csr", "spmv_csr_rows", "stencil", "stencil_temporal", "stencil_sweep", "scale_host", "spmv_csr_host",
    "stencil_host", "SpmvPlan", "mtx_stats", "mtx_read_csr", "matrix_analysis", "fill_uniform", "gen_band_csr", "stencil_init", "load_spec", "load_spec_file", "serialize_spec", "builtin_spec",
    "machine_balance", "tensor_alpha", "attainable", "classify", "ridge_point", "sample_curve", "mem_cmp_ratio", "overlapped_total", "unoverlapped_speedup",
    "kernel_speedup_ceiling", "tensor_core_ceiling", "workload_ceiling", "min_temporal_depth",
    "speedup_bound", "analysis_report",
    "tc_scale_trick_throughput", "fp64_peak_launch", "tuning_set", "kernel_launches",
    "ERROR_KINDS", "EXPORTED_SYMBOLS",
]

CUDA_CORE, TENSOR_CORE = 0, 1          # ExecutionUnit (hardware.hpp:19)
FP64, FP32, FP16 = 0, 1, 2             # Precision (hardware.hpp:21)
MEMORY_BOUND, COMPUTE_BOUND, BALANCED = 0, 1, 2

ERROR_KINDS = [
    "MissingPeak", "ParseError", "ValidationError", "MissingField", "UnknownHardware",
    "InvalidCount", "InvalidIndexSize", "ZeroIntensity", "InvalidAlpha", "ZeroBalance",
    "InvalidRange", "BadBanner", "UnsupportedFormat", "MalformedEntry", "IndexOutOfRange",
    "TruncatedFile", "IoError",
]

_HERE = os.path.dirname(os.path.abspath(__file__))
library_path = os.path.join(_HERE, "librooflens_b200.so")


class RooflensError(RuntimeError):
    """Status code != 0 from the C-ABI.  ``kind`` is the reference ErrorKind
    name (or ``"CudaError"``), ``code`` the raw status."""

    def __init__(self, code: int, message: str):
        super().__init__(message)
        self.code = code
        if 1 <= code <= len(ERROR_KINDS):
            self.kind = ERROR_KINDS[code - 1]
        elif code >= 100:
            self.kind = "CudaError"
        else:
            self.kind = "Error"


class _KChar(C.Structure):
    _fields_ = [("work_flops", C.c_uint64), ("traffic_bytes", C.c_uint64)]


class _HwSpec(C.Structure):
    _fields_ = [("name", C.c_char * 64), ("memory_bandwidth", C.c_double),
                ("l2_cache_bytes", C.c_double), ("peaks", (C.c_double * 3) * 2)]


@dataclass(frozen=True)
class KernelCharacterization:
    """Flattened ``rooflens::KernelCharacterization`` (kernels.hpp:34-44)."""

    work_flops: int
    traffic_bytes: int

    @property
    def intensity(self) -> float:
        return self.work_flops / self.traffic_bytes


@dataclass(frozen=True)
class HardwareSpec:
    """``rooflens::HardwareSpec`` (hardware.hpp:43-58), SI units.  The FP64
    peaks are the positional fields; ``fp32`` / ``fp16`` hold (cuda_core,
    tensor_core) pairs; 0 = no entry (MissingPeak on use)."""

    name: str
    memory_bandwidth: float
    l2_cache_bytes: float
    peak_cuda_core: float
    peak_tensor_core: float = 0.0
    fp32: tuple = (0.0, 0.0)
    fp16: tuple = (0.0, 0.0)

    def peak_table(self):
        """[unit][precision] (rl_unit x rl_precision ordinals)."""
        return ((self.peak_cuda_core, self.fp32[0], self.fp16[0]),
                (self.peak_tensor_core, self.fp32[1], self.fp16[1]))

    def _c(self) -> _HwSpec:
        s = _HwSpec()
        s.name = self.name.encode()[:63]
        s.memory_bandwidth = self.memory_bandwidth
        s.l2_cache_bytes = self.l2_cache_bytes
        for u, row in enumerate(self.peak_table()):
            for p, v in enumerate(row):
                s.peaks[u][p] = v
        return s

    @staticmethod
    def _from(s: _HwSpec) -> "HardwareSpec":
        t = [[s.peaks[u][p] for p in range(3)] for u in range(2)]
        return HardwareSpec(s.name.decode(), s.memory_bandwidth, s.l2_cache_bytes, t[0][0], t[1][0],
                            (t[0][1], t[1][1]), (t[0][2], t[1][2]))


_u64, _i64, _dbl, _int, _ptr = C.c_uint64, C.c_int64, C.c_double, C.c_int, C.c_void_p
_KP = C.POINTER(_KChar)
_HP = C.POINTER(_HwSpec)

# name -> (restype, argtypes); exactly the symbols include/rooflens_b200.h declares.
_SIGNATURES = {
    "rl_last_error": (C.c_char_p, []),
    "rl_version": (C.c_char_p, []),
    "rl_kernel_launches": (_u64, []),
    "rl_scale_model": (_int, [_u64, _int, _KP]),
    "rl_gemv_model": (_int, [_u64, _u64, _int, _KP]),
    "rl_spmv_generic_model": (_int, [_u64, _u64, _u64, _u64, _u64, _u64, _u64, _int, _KP]),
    "rl_spmv_csr_model": (_int, [_u64, _u64, _u64, _u64, _int, _KP]),
    "rl_stencil_model": (_int, [C.c_char_p, _int, _u64, _KP]),
    "rl_stencil_preset": (_int, [C.c_char_p, C.POINTER(_int), C.POINTER(_u64), C.POINTER(_int)]),
    "rl_stencil_default_weights": (_int, [C.c_char_p, C.POINTER(_dbl), _u64]),
    "rl_scale": (_int, [_int, _int, _ptr, _ptr, _dbl, _u64, _ptr, _KP]),
    "rl_gemv": (_int, [_int, _int, _u64, _u64, _ptr, _ptr, _ptr, _ptr, _KP]),
    "rl_spmv_csr": (_int, [_int, _int, _u64, _u64, _u64, _ptr, _ptr, _ptr, _ptr, _ptr, _ptr, _KP]),
    "rl_spmv_csr_rows": (_int, [_int, _int, _u64, _u64, _ptr, _ptr, _ptr, _ptr, _i64, _ptr, _ptr]),
    "rl_stencil": (_int, [_int, _int, C.c_char_p, C.POINTER(_u64), _ptr, _u64, _ptr, _ptr, _ptr, _KP]),
    "rl_stencil_temporal": (_int, [_int, _int, C.c_char_p, C.POINTER(_u64), _ptr, _u64, _u64, _ptr, _ptr,
                                   _ptr, C.POINTER(_int), _KP]),
    "rl_stencil_sweep": (_int, [_int, _int, C.c_char_p, C.POINTER(_u64), _ptr, _u64, _u64, _ptr,
                                _ptr, _ptr]),
    "rl_scale_host": (_int, [_int, _int, _ptr, _ptr, _dbl, _u64, _KP]),
    "rl_spmv_csr_host": (_int, [_int, _int, _u64, _u64, _u64, _ptr, _ptr, _ptr, _ptr, _ptr, _KP]),
    "rl_stencil_host": (_int, [_int, _int, C.c_char_p, C.POINTER(_u64), _ptr, _u64, _ptr, _ptr, _KP]),
    "rl_host_workspace_release": (_int, []),
    "rl_spmv_plan_create": (_int, [_int, _int, _u64, _u64, _u64, _ptr, _ptr, _ptr, C.POINTER(_ptr)]),
    "rl_spmv_plan_execute_host": (_int, [_ptr, _ptr, _ptr, _KP]),
    "rl_spmv_plan_execute_host_async": (_int, [_ptr, _ptr, _ptr, _KP]),
    "rl_spmv_plan_wait": (_int, [_ptr]),
    "rl_spmv_plan_execute": (_int, [_ptr, _ptr, _ptr, _ptr, _KP]),
    "rl_spmv_plan_destroy": (_int, [_ptr]),
    "rl_spmv_plan_info": (_int, [_ptr, C.POINTER(_int), C.POINTER(_u64)]),
    "rl_fill_uniform": (_int, [_ptr, _u64, _u64, _u64, _u64, _int, _ptr]),
    "rl_gen_band_csr": (_int, [_u64, _u64, _u64, C.c_uint32, _u64, _u64, _ptr, _ptr, _ptr, _ptr]),
    "rl_stencil_init": (_int, [_ptr, C.POINTER(_u64), _int, _u64, _u64, _int, _u64, _ptr]),
    "rl_mtx_stats": (_int, [C.c_char_p, C.POINTER(_u64), C.POINTER(_u64), C.POINTER(_u64)]),
    "rl_mtx_read_csr": (_int, [C.c_char_p, _u64, _u64, _ptr, _ptr, _ptr, C.POINTER(_u64), C.POINTER(_u64),
                               C.POINTER(_u64)]),
    "rl_matrix_analysis_of": (_int, [_u64, _u64, _u64, _HP, _int, _ptr]),
    "rl_load_spec": (_int, [C.c_char_p, _HP]),
    "rl_builtin_spec": (_int, [C.c_char_p, _HP]),
    "rl_load_spec_file": (_int, [C.c_char_p, _HP]),
    "rl_serialize_spec": (_int, [_HP, C.c_char_p, _u64, C.POINTER(_u64)]),
    "rl_machine_balance": (_int, [_HP, _int, _int, C.POINTER(_dbl)]),
    "rl_tensor_alpha": (_int, [_HP, _int, C.POINTER(_dbl)]),
    "rl_attainable": (_int, [_HP, _int, _int, _dbl, C.POINTER(_dbl)]),
    "rl_classify": (_int, [_dbl, _dbl]),
    "rl_ridge_point": (_int, [_HP, _int, _int, C.POINTER(_dbl)]),
    "rl_mem_cmp_ratio": (_int, [_dbl, _dbl, C.POINTER(_dbl)]),
    "rl_overlapped_total": (_int, [_dbl, _dbl, _dbl, C.POINTER(_dbl)]),
    "rl_sample_curve": (_int, [_HP, _int, _int, _dbl, _dbl, _u64, _ptr, _ptr, _u64, C.POINTER(_u64)]),
    "rl_unoverlapped_speedup": (_int, [_dbl, _dbl, _dbl, _dbl, C.POINTER(_dbl)]),
    "rl_kernel_speedup_ceiling": (_int, [_dbl, _dbl, _dbl, C.POINTER(_dbl), C.POINTER(_int)]),
    "rl_tensor_core_ceiling": (_int, [_dbl, C.POINTER(_dbl)]),
    "rl_workload_ceiling": (_int, [_dbl, _dbl, C.POINTER(_dbl)]),
    "rl_min_temporal_depth": (_int, [_dbl, _dbl, C.POINTER(_u64)]),
    "rl_tc_scale_trick_throughput": (_int, [_dbl, _u64, _u64, C.POINTER(_dbl)]),
    "rl_bound_kind_name": (C.c_char_p, [_int]),
    "rl_unoverlapped_bound": (_int, [_dbl, _dbl, _dbl, _dbl, _ptr, C.c_char_p, _u64, C.POINTER(_u64)]),
    "rl_kernel_ceiling_bound": (_int, [_dbl, _dbl, _dbl, _ptr, C.c_char_p, _u64, C.POINTER(_u64)]),
    "rl_tensor_core_bound": (_int, [_dbl, _ptr, C.c_char_p, _u64, C.POINTER(_u64)]),
    "rl_workload_bound": (_int, [_dbl, _dbl, _ptr, C.c_char_p, _u64, C.POINTER(_u64)]),
    "rl_analysis_render": (_int, [_HP, _int, C.c_char_p, _u64, _u64, C.POINTER(_dbl), C.POINTER(_dbl), _int,
                                  C.c_char_p, _u64, C.POINTER(_u64)]),
    "rl_fp64_peak_launch": (_int, [_int, _u64, _ptr, _ptr, C.POINTER(_dbl)]),
    "rl_tuning_set": (_int, [C.c_char_p, _i64, C.POINTER(_i64)]),
    # multi-GPU (dist.py wraps these)
    "rl_dist_unique_id": (_int, [_ptr]),
    "rl_dist_init": (_int, [_int, _int, _ptr, C.POINTER(_ptr)]),
    "rl_dist_destroy": (_int, [_ptr]),
    "rl_dist_info": (_int, [_ptr, C.POINTER(_int), C.POINTER(_int), C.POINTER(_int), C.POINTER(_int)]),
    "rl_dist_allreduce_u64": (_int, [_ptr, C.POINTER(_u64)]),
    "rl_dist_allreduce_max": (_int, [_ptr, C.POINTER(_dbl)]),
    "rl_dist_block": (_int, [_u64, _u64, _u64, C.POINTER(_u64), C.POINTER(_u64)]),
    "rl_dist_spmv_part": (_int, [_u64, _u64, _u64, _u64, C.POINTER(_u64), C.POINTER(_u64), C.POINTER(_u64),
                                 C.POINTER(_u64)]),
    "rl_dist_stencil_part": (_int, [C.c_char_p, C.POINTER(_u64), _u64, _u64, C.POINTER(_u64), C.POINTER(_u64),
                                    C.POINTER(_u64), C.POINTER(_u64)]),
    "rl_dist_spmv_schedule": (_int, [_u64, _u64, _int, _int, _int, _ptr, _u64, C.POINTER(_u64)]),
    "rl_dist_stencil_schedule": (_int, [C.c_char_p, C.POINTER(_u64), _int, _int, _int, _ptr, _u64,
                                        C.POINTER(_u64)]),
    "rl_dist_scale": (_int, [_ptr, _int, _int, _ptr, _ptr, _dbl, _u64, _ptr, _KP]),
    "rl_dist_spmv_create": (_int, [_ptr, _int, _int, _u64, _u64, _int, _ptr, _ptr, _ptr, _ptr, _ptr,
                                   C.POINTER(_ptr)]),
    "rl_dist_spmv_execute": (_int, [_ptr, _ptr, _KP]),
    "rl_dist_spmv_destroy": (_int, [_ptr]),
    "rl_dist_stencil_create": (_int, [_ptr, _int, _int, C.c_char_p, C.POINTER(_u64), _ptr, _int, _ptr, _ptr,
                                      C.POINTER(_ptr)]),
    "rl_dist_stencil_run": (_int, [_ptr, _u64, _ptr, C.POINTER(_int), _KP]),
    "rl_dist_stencil_destroy": (_int, [_ptr]),
}
EXPORTED_SYMBOLS = sorted(_SIGNATURES)

_lib: Optional[C.CDLL] = None


def lib() -> C.CDLL:
    """Load the in-tree sm_100a library.  Raises (never falls back) if absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(library_path):
            raise ImportError(
                f"{library_path} is missing: build it with `python -c 'import __graft_entry__ as g; "
                f"g.build()'` (or `make -C paper_2502_16851_b200/csrc`)")
        L = C.CDLL(library_path)
        for name, (res, args) in _SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _check(code: int) -> None:
    if code != 0:
        msg = lib().rl_last_error().decode(errors="replace")
        raise RooflensError(code, msg or f"status {code}")


def _kc(k: _KChar) -> KernelCharacterization:
    return KernelCharacterization(int(k.work_flops), int(k.traffic_bytes))


# ----------------------------------------------------------------------------
# tensor plumbing (torch is only the allocator/stream provider)
# ----------------------------------------------------------------------------
def _dev_ptr(t, dtype_name: str, what: str) -> int:
    import torch

    want = {"f64": torch.float64, "i32": torch.int32}[dtype_name]
    if not isinstance(t, torch.Tensor):
        raise TypeError(f"{what} must be a torch.Tensor")
    if t.dtype != want:
        raise TypeError(f"{what} must be {want}, got {t.dtype}")
    if not t.is_cuda:
        raise ValueError(f"{what} must be a CUDA tensor")
    if not t.is_contiguous():
        raise ValueError(f"{what} must be contiguous")
    return t.data_ptr()


def _host_ptr(a, dtype_name: str, what: str) -> int:
    """numpy array or CPU tensor (pinned for full-speed copies)."""
    try:
        import torch

        if isinstance(a, torch.Tensor):
            want = {"f64": torch.float64, "i32": torch.int32}[dtype_name]
            if a.is_cuda or a.dtype != want or not a.is_contiguous():
                raise ValueError(f"{what} must be a contiguous CPU {want} tensor")
            return a.data_ptr()
    except ImportError:  # pragma: no cover
        pass
    import numpy as np

    want = {"f64": np.float64, "i32": np.int32}[dtype_name]
    if not isinstance(a, np.ndarray) or a.dtype != want or not a.flags["C_CONTIGUOUS"]:
        raise ValueError(f"{what} must be a C-contiguous numpy {want.__name__} array")
    return a.ctypes.data


def _stream(stream) -> int:
    if stream is None:
        import torch

        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


# ----------------------------------------------------------------------------
# accounting (kernels.cpp:74-155)
# ----------------------------------------------------------------------------
def scale_model(n: int, precision: int = FP64) -> KernelCharacterization:
    k = _KChar()
    _check(lib().rl_scale_model(n, precision, C.byref(k)))
    return _kc(k)


def gemv_model(m: int, n: int, precision: int = FP64) -> KernelCharacterization:
    k = _KChar()
    _check(lib().rl_gemv_model(m, n, precision, C.byref(k)))
    return _kc(k)


def spmv_generic_model(rows, cols, nnz, index_entry_count=0, index_entry_bytes=0,
                       packed_entry_count=0, packed_entry_bytes=0, precision=FP64):
    k = _KChar()
    _check(lib().rl_spmv_generic_model(rows, cols, nnz, index_entry_count, index_entry_bytes,
                                       packed_entry_count, packed_entry_bytes, precision,
                                       C.byref(k)))
    return _kc(k)


def spmv_csr_model(rows: int, cols: int, nnz: int, index_bytes: int = 4,
                   precision: int = FP64) -> KernelCharacterization:
    k = _KChar()
    _check(lib().rl_spmv_csr_model(rows, cols, nnz, index_bytes, precision, C.byref(k)))
    return _kc(k)


def stencil_model(preset: str, precision: int = FP64, temporal_depth: int = 1):
    k = _KChar()
    _check(lib().rl_stencil_model(preset.encode(), precision, temporal_depth, C.byref(k)))
    return _kc(k)


def stencil_preset(name: str):
    """(dimensionality, point_count, radius)."""
    d, p, r = _int(), _u64(), _int()
    _check(lib().rl_stencil_preset(name.encode(), C.byref(d), C.byref(p), C.byref(r)))
    return d.value, p.value, r.value


def stencil_default_weights(name: str) -> list:
    buf = (_dbl * 64)()
    _check(lib().rl_stencil_default_weights(name.encode(), buf, 64))
    return list(buf[: stencil_preset(name)[1]])


# ----------------------------------------------------------------------------
# executing kernels (device tensors)
# ----------------------------------------------------------------------------
def scale(a, b, q: float, unit: int = CUDA_CORE, stream=None, precision: int = FP64):
    """a[i] = q * b[i] on the GPU."""
    n = b.numel()
    if a.numel() != n:
        raise ValueError("a and b must have the same number of elements")
    k = _KChar()
    _check(lib().rl_scale(unit, precision, _dev_ptr(a, "f64", "a"), _dev_ptr(b, "f64", "b"),
                          float(q), n, _stream(stream), C.byref(k)))
    return _kc(k)


def gemv(A, x, y, unit: int = CUDA_CORE, stream=None, precision: int = FP64):
    """y = A x for a row-major (m, n) float64 tensor A."""
    m, n = A.shape
    if x.numel() != n or y.numel() != m:
        raise ValueError("inconsistent GEMV sizes")
    k = _KChar()
    _check(lib().rl_gemv(unit, precision, m, n, _dev_ptr(A, "f64", "A"), _dev_ptr(x, "f64", "x"),
                         _dev_ptr(y, "f64", "y"), _stream(stream), C.byref(k)))
    return _kc(k)


def spmv_csr(row_ptr, col, val, x, y, unit: int = CUDA_CORE, stream=None, precision: int = FP64):
    """y = A x for a CSR matrix with int32 indices."""
    m = row_ptr.numel() - 1
    n = x.numel()
    nnz = val.numel()
    if y.numel() != m or col.numel() != nnz:
        raise ValueError("inconsistent CSR / vector sizes")
    k = _KChar()
    _check(lib().rl_spmv_csr(unit, precision, m, n, nnz, _dev_ptr(row_ptr, "i32", "row_ptr"),
                             _dev_ptr(col, "i32", "col") if nnz else None,
                             _dev_ptr(val, "f64", "val") if nnz else None,
                             _dev_ptr(x, "f64", "x"), _dev_ptr(y, "f64", "y"), _stream(stream),
                             C.byref(k)))
    return _kc(k)


def spmv_csr_rows(row_begin: int, row_end: int, row_ptr, col, val, x, y, col_base: int = 0,
                  unit: int = CUDA_CORE, stream=None, precision: int = FP64) -> None:
    """Rows [row_begin, row_end) of y = A x, reading x[col - col_base]."""
    _check(lib().rl_spmv_csr_rows(unit, precision, row_begin, row_end,
                                  _dev_ptr(row_ptr, "i32", "row_ptr"),
                                  _dev_ptr(col, "i32", "col") if col.numel() else None,
                                  _dev_ptr(val, "f64", "val") if val.numel() else None,
                                  _dev_ptr(x, "f64", "x") if x.numel() else None,
                                  col_base, _dev_ptr(y, "f64", "y"), _stream(stream)))


def _dims(preset: str, u) -> "C.Array":
    dim = stencil_preset(preset)[0]
    shape = tuple(u.shape)
    if len(shape) != dim:
        raise ValueError(f"{preset} needs a {dim}-D field, got shape {shape}")
    if dim == 2:
        ny, nx = shape
        return (_u64 * 3)(nx, ny, 1)
    nz, ny, nx = shape
    return (_u64 * 3)(nx, ny, nz)


def _weights(preset: str, weights: Optional[Sequence[float]]):
    if weights is None:
        return None
    npts = stencil_preset(preset)[1]
    if len(weights) != npts:
        raise ValueError(f"{preset} takes {npts} weights, got {len(weights)}")
    return (_dbl * npts)(*[float(w) for w in weights])


def stencil(preset: str, u, v, steps: int, weights=None, unit: int = CUDA_CORE, stream=None,
            precision: int = FP64):
    """`steps` Jacobi sweeps ping-ponging u -> v -> u ...; result in u if steps
    is even, else in v.  Field shapes: (ny, nx) or (nz, ny, nx)."""
    if u.shape != v.shape:
        raise ValueError("u and v must have the same shape")
    k = _KChar()
    w = _weights(preset, weights)
    _check(lib().rl_stencil(unit, precision, preset.encode(), _dims(preset, u),
                            C.cast(w, _ptr) if w is not None else None, steps,
                            _dev_ptr(u, "f64", "u"), _dev_ptr(v, "f64", "v"), _stream(stream),
                            C.byref(k)))
    return _kc(k)


def stencil_temporal(preset: str, u, v, steps: int, temporal_depth: int, weights=None,
                     unit: int = CUDA_CORE, stream=None, precision: int = FP64):
    """Temporal blocking: steps/t fused sweeps of t timesteps.  Returns
    (KernelCharacterization, result_tensor)."""
    if u.shape != v.shape:
        raise ValueError("u and v must have the same shape")
    k, inv = _KChar(), _int()
    w = _weights(preset, weights)
    _check(lib().rl_stencil_temporal(unit, precision, preset.encode(), _dims(preset, u),
                                     C.cast(w, _ptr) if w is not None else None, steps, temporal_depth,
                                     _dev_ptr(u, "f64", "u"), _dev_ptr(v, "f64", "v"), _stream(stream),
                                     C.byref(inv), C.byref(k)))
    return _kc(k), (v if inv.value else u)


def stencil_sweep(preset: str, u, v, o_begin: int, o_end: int, weights=None,
                  unit: int = CUDA_CORE, stream=None, precision: int = FP64) -> None:
    """One sweep v = S(u) over outer indices [o_begin, o_end) (rows / planes)."""
    w = _weights(preset, weights)
    _check(lib().rl_stencil_sweep(unit, precision, preset.encode(), _dims(preset, u),
                                  C.cast(w, _ptr) if w is not None else None, o_begin, o_end,
                                  _dev_ptr(u, "f64", "u"), _dev_ptr(v, "f64", "v"),
                                  _stream(stream)))


# ----------------------------------------------------------------------------
# end to end on host buffers
# ----------------------------------------------------------------------------
def scale_host(a, b, q: float, unit: int = CUDA_CORE, precision: int = FP64):
    k = _KChar()
    n = len(b) if not hasattr(b, "numel") else b.numel()
    _check(lib().rl_scale_host(unit, precision, _host_ptr(a, "f64", "a"), _host_ptr(b, "f64", "b"),
                               float(q), n, C.byref(k)))
    return _kc(k)


def spmv_csr_host(row_ptr, col, val, x, y, unit: int = CUDA_CORE, precision: int = FP64):
    size = (lambda t: t.numel() if hasattr(t, "numel") else t.size)
    m, n, nnz = size(row_ptr) - 1, size(x), size(val)
    k = _KChar()
    _check(lib().rl_spmv_csr_host(unit, precision, m, n, nnz, _host_ptr(row_ptr, "i32", "row_ptr"),
                                  _host_ptr(col, "i32", "col"), _host_ptr(val, "f64", "val"),
                                  _host_ptr(x, "f64", "x"), _host_ptr(y, "f64", "y"), C.byref(k)))
    return _kc(k)


def stencil_host(preset: str, u, v, steps: int, weights=None, unit: int = CUDA_CORE,
                 precision: int = FP64):
    k = _KChar()
    w = _weights(preset, weights)
    _check(lib().rl_stencil_host(unit, precision, preset.encode(), _dims(preset, u),
                                 C.cast(w, _ptr) if w is not None else None, steps,
                                 _host_ptr(u, "f64", "u"), _host_ptr(v, "f64", "v"), C.byref(k)))
    return _kc(k)


class SpmvPlan:
    """CSR matrix uploaded once; execute() moves x in and y out per call
    (rl_spmv_plan_* in the C-ABI).  Host arrays: numpy or (pinned) CPU tensors."""

    def __init__(self, row_ptr, col, val, n_cols: int, unit: int = CUDA_CORE, precision: int = FP64):
        size = (lambda t: t.numel() if hasattr(t, "numel") else t.size)
        self.m, self.n, self.nnz = size(row_ptr) - 1, int(n_cols), size(val)
        h = _ptr()
        _check(lib().rl_spmv_plan_create(unit, precision, self.m, self.n, self.nnz,
                                         _host_ptr(row_ptr, "i32", "row_ptr"), _host_ptr(col, "i32", "col"),
                                         _host_ptr(val, "f64", "val"), C.byref(h)))
        self._h = h

    def execute_host(self, x, y) -> KernelCharacterization:
        k = _KChar()
        _check(lib().rl_spmv_plan_execute_host(self._h, _host_ptr(x, "f64", "x"), _host_ptr(y, "f64", "y"),
                                               C.byref(k)))
        return _kc(k)

    def execute_host_async(self, x, y) -> KernelCharacterization:
        """Enqueue one execute_host and return: x must stay unchanged and y
        unread until wait(); consecutive calls overlap on three buffer slots."""
        k = _KChar()
        _check(lib().rl_spmv_plan_execute_host_async(self._h, _host_ptr(x, "f64", "x"), _host_ptr(y, "f64", "y"),
                                                     C.byref(k)))
        return _kc(k)

    def wait(self) -> None:
        _check(lib().rl_spmv_plan_wait(self._h))

    def execute(self, x, y, stream=None) -> KernelCharacterization:
        k = _KChar()
        _check(lib().rl_spmv_plan_execute(self._h, _dev_ptr(x, "f64", "x"), _dev_ptr(y, "f64", "y"),
                                          _stream(stream), C.byref(k)))
        return _kc(k)

    def info(self):
        """(layout, layout_bytes): the layout name and the bytes one execute
        streams for A."""
        t, b = _int(), _u64()
        _check(lib().rl_spmv_plan_info(self._h, C.byref(t), C.byref(b)))
        return self.layout(), int(b.value)

    def layout(self) -> str:
        """"csr" or "colsort" (column-sorted row blocks, spmv_colsort.cu)."""
        t = _int()
        _check(lib().rl_spmv_plan_info(self._h, C.byref(t), None))
        return {0: "csr", 4: "colsort"}[t.value]

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            lib().rl_spmv_plan_destroy(self._h)
            self._h = _ptr()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ----------------------------------------------------------------------------
# generators (device, bit-identical to oracle/oracle.c)
# ----------------------------------------------------------------------------
def fill_uniform(out, seed: int, stream_id: int, idx0: int = 0, kind: int = 0, stream=None):
    _check(lib().rl_fill_uniform(_dev_ptr(out, "f64", "out"), out.numel(), seed, stream_id, idx0,
                                 kind, _stream(stream)))


def gen_band_csr(m_local: int, row0: int, n: int, k: int, hb: int, seed: int, row_ptr, col, val,
                 stream=None):
    _check(lib().rl_gen_band_csr(m_local, row0, n, k, hb, seed,
                                 _dev_ptr(row_ptr, "i32", "row_ptr"), _dev_ptr(col, "i32", "col"),
                                 _dev_ptr(val, "f64", "val"), _stream(stream)))


def stencil_init(u, radius: int, seed: int, outer_begin: int = 0, global_shape=None,
                 stream=None):
    """Fill u (shape (ny, nx) or (nz, ny, nx)) with the BASELINE initial field.
    With global_shape, u is the slab of outer indices [outer_begin,
    outer_begin + u.shape[0]) of that global grid."""
    gs = tuple(global_shape or u.shape)
    dim = len(gs)
    dims = (_u64 * 3)(gs[-1], gs[-2], gs[0] if dim == 3 else 1)
    _check(lib().rl_stencil_init(_dev_ptr(u, "f64", "u"), dims, dim, outer_begin,
                                 outer_begin + u.shape[0], radius, seed, _stream(stream)))


# ----------------------------------------------------------------------------
# Matrix Market
# ----------------------------------------------------------------------------
class _MatrixAnalysis(C.Structure):
    _fields_ = [("work_flops", C.c_uint64), ("traffic_bytes", C.c_uint64), ("boundedness", C.c_int),
                ("kernel_ceiling", C.c_double), ("kernel_ceiling_warnings", C.c_int),
                ("workload_ceiling", C.c_double), ("csr_bytes", C.c_uint64), ("fits_in_l2", C.c_int)]


def mtx_stats(path: str):
    """(rows, cols, expanded nnz) -- reference parse_stats_file semantics."""
    r, c, n = _u64(), _u64(), _u64()
    _check(lib().rl_mtx_stats(os.fsencode(path), C.byref(r), C.byref(c), C.byref(n)))
    return r.value, c.value, n.value


def mtx_read_csr(path: str):
    """CSR (row_ptr int32, col int32, val float64) and the column count."""
    import numpy as np

    rows, cols, nnz = mtx_stats(path)
    rp = np.empty(rows + 1, np.int32)
    col = np.empty(max(nnz, 1), np.int32)
    val = np.empty(max(nnz, 1), np.float64)
    r, c, n = _u64(), _u64(), _u64()
    _check(lib().rl_mtx_read_csr(os.fsencode(path), rows + 1, nnz, rp.ctypes.data, col.ctypes.data,
                                 val.ctypes.data, C.byref(r), C.byref(c), C.byref(n)))
    return rp, col[:nnz], val[:nnz], cols


def matrix_analysis(rows: int, cols: int, nnz: int, spec: HardwareSpec, precision: int = FP64) -> dict:
    """reference stats_to_report (matrix_market.cpp:203-216)."""
    out = _MatrixAnalysis()
    s = spec._c()
    _check(lib().rl_matrix_analysis_of(rows, cols, nnz, C.byref(s), precision, C.byref(out)))
    return {f: getattr(out, f) for f, _ in _MatrixAnalysis._fields_}


# ----------------------------------------------------------------------------
# hardware spec, roofline, bounds
# ----------------------------------------------------------------------------
def load_spec(text: str) -> HardwareSpec:
    s = _HwSpec()
    _check(lib().rl_load_spec(text.encode(), C.byref(s)))
    return HardwareSpec._from(s)


def load_spec_file(path) -> HardwareSpec:
    """reference load_spec_file (hardware.cpp:239-247)."""
    s = _HwSpec()
    _check(lib().rl_load_spec_file(os.fsencode(path), C.byref(s)))
    return HardwareSpec._from(s)


def serialize_spec(spec: HardwareSpec) -> str:
    """reference serialize_spec (hardware.cpp:249-264), byte for byte."""
    s = spec._c()
    n = _u64()
    _check(lib().rl_serialize_spec(C.byref(s), None, 0, C.byref(n)))
    buf = C.create_string_buffer(n.value + 1)
    _check(lib().rl_serialize_spec(C.byref(s), buf, n.value + 1, None))
    return buf.value.decode()


def builtin_spec(name: str) -> HardwareSpec:
    s = _HwSpec()
    _check(lib().rl_builtin_spec(name.encode(), C.byref(s)))
    return HardwareSpec._from(s)


def _d1(fn, *args) -> float:
    out = _dbl()
    _check(fn(*args, C.byref(out)))
    return out.value


def machine_balance(spec: HardwareSpec, unit: int = CUDA_CORE, precision: int = FP64) -> float:
    s = spec._c()
    return _d1(lib().rl_machine_balance, C.byref(s), unit, precision)


def tensor_alpha(spec: HardwareSpec, precision: int = FP64) -> float:
    s = spec._c()
    return _d1(lib().rl_tensor_alpha, C.byref(s), precision)


def attainable(spec: HardwareSpec, intensity: float, unit: int = CUDA_CORE,
               precision: int = FP64) -> float:
    s = spec._c()
    return _d1(lib().rl_attainable, C.byref(s), unit, precision, float(intensity))


def classify(intensity: float, balance: float) -> int:
    return lib().rl_classify(float(intensity), float(balance))


def ridge_point(spec: HardwareSpec, unit: int = CUDA_CORE, precision: int = FP64) -> float:
    s = spec._c()
    return _d1(lib().rl_ridge_point, C.byref(s), unit, precision)


def sample_curve(spec: HardwareSpec, i_min: float, i_max: float, n_points: int, unit: int = CUDA_CORE,
                 precision: int = FP64):
    """[(intensity, attainable)] as the reference's sample_curve (roofline.cpp:40-79)."""
    import numpy as np

    s = spec._c()
    cap = int(n_points) + 1
    xs = np.empty(cap, np.float64)
    ys = np.empty(cap, np.float64)
    cnt = _u64()
    _check(lib().rl_sample_curve(C.byref(s), unit, precision, float(i_min), float(i_max), int(n_points),
                                 xs.ctypes.data, ys.ctypes.data, cap, C.byref(cnt)))
    return list(zip(xs[:cnt.value].tolist(), ys[:cnt.value].tolist()))


def mem_cmp_ratio(balance, intensity) -> float:
    return _d1(lib().rl_mem_cmp_ratio, float(balance), float(intensity))


def overlapped_total(t_cmp, t_mem, t_others) -> float:
    return _d1(lib().rl_overlapped_total, float(t_cmp), float(t_mem), float(t_others))


def unoverlapped_speedup(t_cmp, t_mem, t_others, alpha) -> float:
    return _d1(lib().rl_unoverlapped_speedup, float(t_cmp), float(t_mem), float(t_others),
               float(alpha))


def kernel_speedup_ceiling(alpha, balance, intensity):
    """(value, n_warnings)."""
    out, nw = _dbl(), _int()
    _check(lib().rl_kernel_speedup_ceiling(float(alpha), float(balance), float(intensity),
                                           C.byref(out), C.byref(nw)))
    return out.value, nw.value


def tensor_core_ceiling(alpha) -> float:
    return _d1(lib().rl_tensor_core_ceiling, float(alpha))


def workload_ceiling(intensity, balance) -> float:
    return _d1(lib().rl_workload_ceiling, float(intensity), float(balance))


def min_temporal_depth(balance, single_step_intensity) -> int:
    out = _u64()
    _check(lib().rl_min_temporal_depth(float(balance), float(single_step_intensity), C.byref(out)))
    return int(out.value)


def tc_scale_trick_throughput(peak_tc, m, n) -> float:
    return _d1(lib().rl_tc_scale_trick_throughput, float(peak_tc), int(m), int(n))


class _SpeedupBound(C.Structure):
    _fields_ = [("value", C.c_double), ("kind", C.c_int), ("n_assumptions", C.c_int),
                ("n_warnings", C.c_int)]


BOUND_FUNCS = {"unoverlapped": "rl_unoverlapped_bound", "kernel": "rl_kernel_ceiling_bound",
               "tensor_core": "rl_tensor_core_bound", "workload": "rl_workload_bound"}


def speedup_bound(which: str, *args) -> dict:
    """A reportable SpeedupBound (bounds.hpp:27-45): which = unoverlapped
    (t_cmp, t_mem, t_others, alpha) | kernel (alpha, balance, intensity) |
    tensor_core (alpha) | workload (intensity, balance).  Returns
    {value, kind, kind_name, assumptions, warnings}."""
    fn = getattr(lib(), BOUND_FUNCS[which])
    b, n = _SpeedupBound(), _u64()
    fargs = [float(a) for a in args]
    _check(fn(*fargs, C.byref(b), None, 0, C.byref(n)))
    buf = C.create_string_buffer(n.value + 1)
    _check(fn(*fargs, C.byref(b), buf, n.value + 1, None))
    lines = buf.value.decode().split("\n")[:-1]
    return {"value": b.value, "kind": b.kind, "kind_name": lib().rl_bound_kind_name(b.kind).decode(),
            "assumptions": lines[:b.n_assumptions], "warnings": lines[b.n_assumptions:]}


REPORT_FORMATS = {"text": 0, "json": 1, "csv": 2}


def analysis_report(spec: HardwareSpec, kernel_name: str, kc: KernelCharacterization, fmt: str = "text",
                    balance_override=None, single_step_intensity=None, precision: int = FP64) -> str:
    """rooflens::build_analysis + render_text/json/csv (report.hpp:19-48)
    through rl_analysis_render."""
    s = spec._c()
    bo = C.byref(_dbl(balance_override)) if balance_override is not None else None
    si = C.byref(_dbl(single_step_intensity)) if single_step_intensity is not None else None
    args = (C.byref(s), precision, kernel_name.encode(), int(kc.work_flops), int(kc.traffic_bytes), bo, si,
            REPORT_FORMATS[fmt])
    n = _u64()
    _check(lib().rl_analysis_render(*args, None, 0, C.byref(n)))
    buf = C.create_string_buffer(n.value + 1)
    _check(lib().rl_analysis_render(*args, buf, n.value + 1, None))
    return buf.value.decode()


# ----------------------------------------------------------------------------
# microbenchmarks, knobs, evidence
# ----------------------------------------------------------------------------
def fp64_peak_launch(unit: int, iters: int, sink, stream=None) -> float:
    """Launch the K11 DFMA/DMMA chain kernel; returns its exact flop count."""
    fl = _dbl()
    _check(lib().rl_fp64_peak_launch(unit, iters, _stream(stream), _dev_ptr(sink, "f64", "sink"),
                                     C.byref(fl)))
    return fl.value


def tuning_set(key: str, value: int) -> int:
    prev = _i64()
    _check(lib().rl_tuning_set(key.encode(), int(value), C.byref(prev)))
    return prev.value


def kernel_launches() -> int:
    return int(lib().rl_kernel_launches())
