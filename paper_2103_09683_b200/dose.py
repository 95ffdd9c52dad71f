"""Host-side mirror of the reference's dose API over the C-ABI library ``libdosegpu.so``.

Reference interface mirrored (paths relative to /root/reference/proj):

* ``spmv_rowchunk(m, x, cfg)``  <- ``ddm::spmv_rowchunk`` (include/ddm/spmv.hpp:37, src/spmv.cpp:98-111)
* ``spmv_oracle(m, x)``         <- ``ddm::spmv_oracle`` (spmv.hpp:29, spmv.cpp:82-96) == rowchunk with
                                   lane_width 1, evaluated on the device
* ``RowChunkConfig``            <- ``ddm::RowChunkConfig`` (spmv.hpp:15-18); ``workers`` is accepted
                                   and, as in the reference, never changes a bit of the output
* ``CsrMatrix``                 <- ``ddm::CsrMatrix`` (sparse.hpp:93-108)
* ``Error`` / ``Errc``          <- ``ddm::Error`` / ``ddm::Errc`` (include/ddm/error.hpp:8-41)
* ``checksum_bits``             <- ``ddm::checksum_bits`` (include/ddm/checksum.hpp:25-35)
* ``traffic_bytes``             <- ``ddm::traffic(dims_of(m), layout_of(m)).total_bytes()``
                                   (src/perf_model.cpp:41-54)

Everything numeric runs in CUDA kernels inside libdosegpu.so; there is no CPU fallback, and
importing this module raises when the library is missing.
"""
from __future__ import annotations

import ctypes as C
import enum
import os
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libdosegpu.so")

HALF, SINGLE, DOUBLE = 0, 1, 2          # ddm::ValuePrecision
U16, U32 = 0, 1                         # ddm::IndexWidth
ACCUM_EXACT, ACCUM_FP32 = 0, 1
X_ON_DEVICE, Y_ON_DEVICE, NO_SYNC, PROFILE = 1, 2, 4, 8
_VDTYPE = {HALF: np.uint16, SINGLE: np.float32, DOUBLE: np.float64}


class Errc(enum.IntEnum):
    """ddm::Errc (error.hpp:8-25); status code = 1 + value."""
    DuplicateEntry = 0
    IndexOverflow = 1
    ValueOverflow = 2
    NanInput = 3
    DimensionMismatch = 4
    InvalidConfig = 5
    ZeroTraffic = 6
    ZeroDuration = 7
    BadMagic = 8
    TruncatedFile = 9
    ValidationFailure = 10
    UnsupportedVersion = 11
    ParseError = 12
    UnsupportedFeature = 13
    InconsistentProfile = 14
    IoFailure = 15


class Error(RuntimeError):
    """ddm::Error: carries the status; ``code`` is the Errc for contract errors, else None."""

    def __init__(self, status: int, what: str = ""):
        self.status = status
        self.code: Optional[Errc] = Errc(status - 1) if 1 <= status <= 16 else None
        name = _lib().dg_strerror(status).decode() if _LIB is not None else str(status)
        if status >= 1000:
            name += f" (cudaError {status - 1000})"
        super().__init__(f"{name}: {what}" if what else name)


# ---------------------------------------------------------------- ctypes plumbing ---------
class _View(C.Structure):
    _fields_ = [("rows", C.c_uint64), ("cols", C.c_uint64), ("nnz", C.c_uint64),
                ("value_precision", C.c_uint8), ("index_bytes", C.c_uint8),
                ("col_storage_bytes", C.c_uint8), ("on_device", C.c_uint8),
                ("row_ptr", C.c_void_p), ("col_indices", C.c_void_p), ("values", C.c_void_p)]


class _Options(C.Structure):
    _fields_ = [("struct_size", C.c_uint32), ("device", C.c_int32), ("lane_width", C.c_uint32),
                ("accumulation", C.c_uint32), ("row_begin", C.c_uint64), ("row_end", C.c_uint64)]


class _Profile(C.Structure):
    _fields_ = [("rows", C.c_uint64), ("cols", C.c_uint64),
                ("target_nnz_ratio", C.c_double), ("empty_row_fraction", C.c_double),
                ("row_length_log_mean", C.c_double), ("row_length_log_sigma", C.c_double),
                ("locality_window", C.c_uint64), ("seed", C.c_uint64)]


class _Info(C.Structure):
    _fields_ = [("rows", C.c_uint64), ("cols", C.c_uint64), ("nnz", C.c_uint64),
                ("row_begin", C.c_uint64), ("row_end", C.c_uint64),
                ("value_bytes", C.c_uint32), ("index_bytes", C.c_uint32),
                ("lane_width", C.c_uint32), ("accumulation", C.c_uint32),
                ("device_bytes", C.c_uint64), ("model_bytes", C.c_uint64),
                ("nonempty_rows", C.c_uint64), ("n_kernels", C.c_uint32), ("device", C.c_int32),
                ("read_ns", C.c_uint64)]


class _Timing(C.Structure):
    _fields_ = [("ms_h2d", C.c_float), ("ms_kernels", C.c_float), ("ms_d2h", C.c_float),
                ("ms_total", C.c_float)]


class _KernelTime(C.Structure):
    _fields_ = [("name", C.c_char * 48), ("ms", C.c_float), ("bytes", C.c_uint64),
                ("rows", C.c_uint64), ("nnz", C.c_uint64)]


MAX_DEVICES = 16
GATHER_NONE, GATHER_PEER, GATHER_NCCL = 0, 1, 2


class _MultiOptions(C.Structure):
    _fields_ = [("struct_size", C.c_uint32), ("n_devices", C.c_uint32),
                ("devices", C.c_int32 * MAX_DEVICES), ("lane_width", C.c_uint32),
                ("accumulation", C.c_uint32), ("gather", C.c_uint32)]


_LIB: Optional[C.CDLL] = None

# name -> (restype, argtypes); the exported surface of include/dosegpu.h
_SIGS = {
    "dg_default_options": (None, [C.POINTER(_Options)]),
    "dg_create": (C.c_int, [C.POINTER(_View), C.POINTER(_Options), C.POINTER(C.c_void_p)]),
    "dg_create_generated": (C.c_int, [C.POINTER(_Profile), C.c_uint32, C.c_uint32,
                                      C.POINTER(_Options), C.POINTER(C.c_void_p)]),
    "dg_generated_row_lengths": (C.c_int, [C.POINTER(_Profile), C.c_uint32, C.c_uint64,
                                           C.c_uint64, C.c_int32, C.c_void_p]),
    "dg_create_from_ddm": (C.c_int, [C.c_char_p, C.POINTER(_Options), C.POINTER(C.c_void_p)]),
    "dg_destroy": (C.c_int, [C.c_void_p]),
    "dg_scatter_create": (C.c_int, [C.POINTER(_View), C.c_uint32, C.c_int32, C.POINTER(C.c_void_p)]),
    "dg_scatter_dose": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint32,
                                  C.c_void_p]),
    "dg_scatter_destroy": (C.c_int, [C.c_void_p]),
    "dg_dose": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint32, C.c_void_p]),
    "dg_get_info": (C.c_int, [C.c_void_p, C.POINTER(_Info)]),
    "dg_last_timing": (C.c_int, [C.c_void_p, C.POINTER(_Timing)]),
    "dg_copy_rows": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint64, C.c_void_p, C.c_void_p,
                               C.c_void_p]),
    "dg_copy_row_ptr": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint64, C.c_void_p]),
    "dg_checksum_bits": (C.c_int, [C.c_void_p, C.c_uint64, C.c_int, C.POINTER(C.c_uint64)]),
    "dg_traffic_bytes": (C.c_uint64, [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint32, C.c_uint32]),
    "dg_partition_rows": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint32, C.c_uint32, C.c_void_p]),
    "dg_partition_lengths": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint32, C.c_uint32, C.c_void_p]),
    "dg_kernel_times": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint32, C.POINTER(C.c_uint32)]),
    "dg_debug_trace": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.POINTER(C.c_uint64)]),
    "dg_seeded_vector": (None, [C.c_uint64, C.c_uint64, C.c_void_p]),
    "dg_set_gather_targets": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p), C.c_uint32]),
    "dg_set_block_targets": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p), C.c_uint32]),
    "dg_ipc_alloc": (C.c_int, [C.c_uint64, C.c_int32, C.POINTER(C.c_void_p), C.c_void_p]),
    "dg_ipc_open": (C.c_int, [C.c_void_p, C.c_int32, C.POINTER(C.c_void_p)]),
    "dg_ipc_close": (C.c_int, [C.c_void_p]),
    "dg_ipc_free": (C.c_int, [C.c_void_p]),
    "dg_multi_default_options": (None, [C.POINTER(_MultiOptions)]),
    "dg_multi_create": (C.c_int, [C.POINTER(_View), C.POINTER(_MultiOptions), C.POINTER(C.c_void_p)]),
    "dg_multi_create_generated": (C.c_int, [C.POINTER(_Profile), C.c_uint32, C.c_uint32,
                                            C.POINTER(_MultiOptions), C.POINTER(C.c_void_p)]),
    "dg_multi_dose": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint32]),
    "dg_multi_bounds": (C.c_int, [C.c_void_p, C.POINTER(C.c_uint32), C.c_void_p]),
    "dg_multi_shard": (C.c_int, [C.c_void_p, C.c_uint32, C.POINTER(C.c_void_p)]),
    "dg_multi_device_d": (C.c_int, [C.c_void_p, C.c_uint32, C.POINTER(C.c_void_p),
                                    C.POINTER(C.c_void_p)]),
    "dg_multi_last_timing": (C.c_int, [C.c_void_p, C.POINTER(_Timing)]),
    "dg_multi_destroy": (C.c_int, [C.c_void_p]),
    "dg_strerror": (C.c_char_p, [C.c_int]),
    "dg_version": (C.c_char_p, []),
}


def _lib() -> C.CDLL:
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing -- build it with "
                              "`python -c 'import __graft_entry__ as g; g.build()'` "
                              "(there is no CPU fallback)")
        lib = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            f = getattr(lib, name)
            f.restype = res
            f.argtypes = args
        _LIB = lib
    return _LIB


def _check(status: int, what: str = "") -> None:
    if status != 0:
        raise Error(status, what)


# ---------------------------------------------------------------- the data model ----------
@dataclass
class CsrMatrix:
    """ddm::CsrMatrix (sparse.hpp:93-108): u64 row_ptr, u32 col_indices in memory whatever the
    ``index_width`` tag, values as bit patterns of ``precision``."""
    rows: int
    cols: int
    index_width: int
    row_ptr: np.ndarray
    col_indices: np.ndarray
    values: np.ndarray
    precision: int = HALF

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1]) if len(self.row_ptr) else 0


@dataclass
class RowChunkConfig:
    """ddm::RowChunkConfig (spmv.hpp:15-18)."""
    lane_width: int = 32
    workers: int = 1


@dataclass
class Profile:
    """ddm::MatrixProfile (matgen.hpp:18-27)."""
    rows: int
    cols: int
    target_nnz_ratio: float
    empty_row_fraction: float
    row_length_log_mean: float
    row_length_log_sigma: float
    locality_window: int
    seed: int

    def _c(self) -> _Profile:
        return _Profile(self.rows, self.cols, self.target_nnz_ratio, self.empty_row_fraction,
                        self.row_length_log_mean, self.row_length_log_sigma,
                        self.locality_window, self.seed)


def _profiles(p) -> tuple:
    ps = [p] if isinstance(p, Profile) else list(p)
    arr = (_Profile * len(ps))(*[q._c() for q in ps])
    return arr, len(ps)


def _options(device: int, lane_width: int, accumulation: int, row_begin: int, row_end: int):
    o = _Options()
    _lib().dg_default_options(C.byref(o))
    o.device, o.lane_width, o.accumulation = device, lane_width, accumulation
    o.row_begin, o.row_end = row_begin, row_end
    return o


# ---------------------------------------------------------------- the engine --------------
class DoseEngine:
    """A matrix resident on one GPU (the whole matrix, or a row shard of it).

    Create once (validation, row plan, native-encoding upload), then ``dose(x)`` as often as the
    optimisation loop needs -- the reference pays these costs inside every spmv_rowchunk call.
    """

    def __init__(self, handle: C.c_void_p):
        self._h = handle
        info = _Info()
        _check(_lib().dg_get_info(self._h, C.byref(info)), "dg_get_info")
        self.info = {k: getattr(info, k) for k, _ in _Info._fields_}

    # --- constructors ---------------------------------------------------------------------
    @classmethod
    def from_csr(cls, m: CsrMatrix, *, lane_width: int = 32, accumulation: int = ACCUM_EXACT,
                 device: int = -1, row_begin: int = 0, row_end: int = 0) -> "DoseEngine":
        rp = np.ascontiguousarray(m.row_ptr, dtype=np.uint64)
        if m.col_indices.dtype == np.uint16:
            col, csb = np.ascontiguousarray(m.col_indices), 2
        else:
            col, csb = np.ascontiguousarray(m.col_indices, dtype=np.uint32), 4
        val = np.ascontiguousarray(m.values, dtype=_VDTYPE[m.precision])
        view = _View(m.rows, m.cols, m.nnz, m.precision, 2 if m.index_width == U16 else 4, csb, 0,
                     rp.ctypes.data, col.ctypes.data, val.ctypes.data)
        h = C.c_void_p()
        opts = _options(device, lane_width, accumulation, row_begin, row_end)
        _check(_lib().dg_create(C.byref(view), C.byref(opts), C.byref(h)), "dg_create")
        return cls(h)

    @classmethod
    def from_device_arrays(cls, rows: int, cols: int, nnz: int, precision: int, index_bytes: int,
                           row_ptr_ptr: int, col_ptr: int, col_storage_bytes: int, val_ptr: int,
                           **kw) -> "DoseEngine":
        view = _View(rows, cols, nnz, precision, index_bytes, col_storage_bytes, 1, row_ptr_ptr,
                     col_ptr, val_ptr)
        h = C.c_void_p()
        opts = _options(kw.get("device", -1), kw.get("lane_width", 32),
                        kw.get("accumulation", ACCUM_EXACT), kw.get("row_begin", 0),
                        kw.get("row_end", 0))
        _check(_lib().dg_create(C.byref(view), C.byref(opts), C.byref(h)), "dg_create")
        return cls(h)

    @classmethod
    def from_ddm(cls, path: str, *, lane_width: int = 32, accumulation: int = ACCUM_EXACT,
                 device: int = -1, row_begin: int = 0, row_end: int = 0) -> "DoseEngine":
        """A DDM1 file (ddm::read_ddm's container) streamed straight into device memory."""
        h = C.c_void_p()
        opts = _options(device, lane_width, accumulation, row_begin, row_end)
        _check(_lib().dg_create_from_ddm(os.fsencode(path), C.byref(opts), C.byref(h)),
               "dg_create_from_ddm")
        return cls(h)

    @classmethod
    def generate(cls, profiles, *, index_bytes: int = 0, lane_width: int = 32,
                 accumulation: int = ACCUM_EXACT, device: int = -1, row_begin: int = 0,
                 row_end: int = 0) -> "DoseEngine":
        arr, n = _profiles(profiles)
        h = C.c_void_p()
        opts = _options(device, lane_width, accumulation, row_begin, row_end)
        _check(_lib().dg_create_generated(arr, n, index_bytes, C.byref(opts), C.byref(h)),
               "dg_create_generated")
        return cls(h)

    # --- the dose -------------------------------------------------------------------------
    def dose(self, x: np.ndarray, out: Optional[np.ndarray] = None) -> np.ndarray:
        """d = A.x with host arrays (H2D x, kernels, D2H d)."""
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = _out_array(out, self.info["rows"])
        _check(_lib().dg_dose(self._h, x.ctypes.data, len(x), y.ctypes.data, 0, None), "dg_dose")
        return y

    def dose_device(self, x_ptr: int, x_len: int, y_ptr: int, stream: int = 0,
                    sync: bool = True, profile: bool = False) -> None:
        """d = A.x with device-resident x / y (raw pointers, e.g. torch.Tensor.data_ptr())."""
        flags = X_ON_DEVICE | Y_ON_DEVICE | (0 if sync else NO_SYNC) | (PROFILE if profile else 0)
        _check(_lib().dg_dose(self._h, C.c_void_p(x_ptr), x_len, C.c_void_p(y_ptr), flags,
                              C.c_void_p(stream) if stream else None), "dg_dose")

    def dose_host_ptrs(self, x_ptr: int, x_len: int, y_ptr: int, stream: int = 0) -> None:
        """d = A.x from (pinned) host pointers -- the end-to-end path."""
        _check(_lib().dg_dose(self._h, C.c_void_p(x_ptr), x_len, C.c_void_p(y_ptr), 0,
                              C.c_void_p(stream) if stream else None), "dg_dose")

    def set_gather_targets(self, ptrs: Sequence[int]) -> None:
        """Fused d gather: every later dose also writes its rows, at their global row index, into
        each of these full-d device buffers (this rank's own and its peers' IPC mappings)."""
        arr = (C.c_void_p * max(len(ptrs), 1))(*[C.c_void_p(p) for p in ptrs])
        _check(_lib().dg_set_gather_targets(self._h, arr, len(ptrs)), "dg_set_gather_targets")

    def set_block_targets(self, ptrs: Sequence[int]) -> None:
        """The d gather by the copy engines: every later dose copies its rows, row block by row
        block as the tile kernel finishes each block, into each of these full-d device buffers
        (at their global row index)."""
        arr = (C.c_void_p * max(len(ptrs), 1))(*[C.c_void_p(p) for p in ptrs])
        _check(_lib().dg_set_block_targets(self._h, arr, len(ptrs)), "dg_set_block_targets")

    def kernel_times(self) -> list:
        """Per-launch CUDA-event times + algorithmic bytes of the last profiled dose."""
        buf = (_KernelTime * 16)()
        n = C.c_uint32()
        _check(_lib().dg_kernel_times(self._h, buf, 16, C.byref(n)), "dg_kernel_times")
        return [{"name": buf[i].name.decode(), "ms": buf[i].ms, "bytes": buf[i].bytes,
                 "rows": buf[i].rows, "nnz": buf[i].nnz} for i in range(n.value)]

    def debug_trace(self) -> np.ndarray:
        """The DG_TRACE timeline of the last dose (uint64 words, see dg_debug_trace); empty when
        the handle was created without DG_TRACE."""
        cap = 4 * 1024 + 3 * 1_000_000
        buf = np.zeros(cap, dtype=np.uint64)
        n = C.c_uint64()
        _check(_lib().dg_debug_trace(self._h, buf.ctypes.data, cap, C.byref(n)), "dg_debug_trace")
        return buf[:n.value].copy()

    def last_timing(self) -> dict:
        t = _Timing()
        _check(_lib().dg_last_timing(self._h, C.byref(t)), "dg_last_timing")
        return {"ms_h2d": t.ms_h2d, "ms_kernels": t.ms_kernels, "ms_d2h": t.ms_d2h,
                "ms_total": t.ms_total}

    def row_ptr(self, r0: int = 0, r1: Optional[int] = None) -> np.ndarray:
        """Shard row pointers [r0, r1] (not rebased)."""
        r1 = self.info["rows"] if r1 is None else r1
        rp = np.empty(r1 - r0 + 1, dtype=np.uint64)
        _check(_lib().dg_copy_row_ptr(self._h, r0, r1, rp.ctypes.data), "dg_copy_row_ptr")
        return rp

    def copy_rows(self, r0: int, r1: int) -> CsrMatrix:
        """Rows [r0, r1) of the resident shard back in the reference's host encoding
        (u32 column indices in memory, value bit patterns)."""
        ends = self.row_ptr(r0, r1)
        n = int(ends[-1] - ends[0])
        prec = {2: HALF, 4: SINGLE, 8: DOUBLE}[self.info["value_bytes"]]
        rp = np.empty(r1 - r0 + 1, dtype=np.uint64)
        col = np.empty(max(n, 1), dtype=np.uint32)
        val = np.empty(max(n, 1), dtype=_VDTYPE[prec])
        _check(_lib().dg_copy_rows(self._h, r0, r1, rp.ctypes.data, col.ctypes.data,
                                   val.ctypes.data), "dg_copy_rows")
        return CsrMatrix(r1 - r0, self.info["cols"], U16 if self.info["index_bytes"] == 2 else U32,
                         rp, col[:n], val[:n], prec)

    def close(self) -> None:
        if self._h:
            if getattr(self, "_owner", True):
                _lib().dg_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


class MultiDoseEngine:
    """One process, several GPUs behind one handle (dg_multi_*): the rows cut into nnz-balanced
    shards, one per entry of ``devices`` (a device may repeat: virtual shards), doses run
    concurrently and the d slices are gathered per ``gather`` (GATHER_NONE / GATHER_PEER /
    GATHER_NCCL).  The reference's own fan-out, ddm::spmv_rowchunk -> parallel_blocks
    (spmv.hpp:37, spmv.cpp:17-32), behind one call."""

    def __init__(self, handle: C.c_void_p):
        self._h = handle
        n = C.c_uint32()
        _check(_lib().dg_multi_bounds(self._h, C.byref(n), None), "dg_multi_bounds")
        b = np.empty(n.value + 1, dtype=np.uint64)
        _check(_lib().dg_multi_bounds(self._h, C.byref(n), b.ctypes.data), "dg_multi_bounds")
        self.bounds = b
        self.rows = int(b[-1])
        self.n_shards = n.value
        sh = C.c_void_p()
        _check(_lib().dg_multi_shard(self._h, 0, C.byref(sh)), "dg_multi_shard")
        info = _Info()
        _check(_lib().dg_get_info(sh, C.byref(info)), "dg_get_info")
        self.cols = info.cols

    @staticmethod
    def _opts(devices, lane_width, accumulation, gather) -> _MultiOptions:
        if not 1 <= len(devices) <= MAX_DEVICES:
            raise Error(1 + Errc.InvalidConfig, f"1..{MAX_DEVICES} devices")
        o = _MultiOptions()
        _lib().dg_multi_default_options(C.byref(o))
        o.n_devices = len(devices)
        for i, d in enumerate(devices):
            o.devices[i] = int(d)
        o.lane_width, o.accumulation, o.gather = lane_width, accumulation, gather
        return o

    @classmethod
    def from_csr(cls, m: CsrMatrix, devices: Sequence[int], *, gather: int = GATHER_PEER,
                 lane_width: int = 32, accumulation: int = ACCUM_EXACT) -> "MultiDoseEngine":
        rp = np.ascontiguousarray(m.row_ptr, dtype=np.uint64)
        if m.col_indices.dtype == np.uint16:
            col, csb = np.ascontiguousarray(m.col_indices), 2
        else:
            col, csb = np.ascontiguousarray(m.col_indices, dtype=np.uint32), 4
        val = np.ascontiguousarray(m.values, dtype=_VDTYPE[m.precision])
        view = _View(m.rows, m.cols, m.nnz, m.precision, 2 if m.index_width == U16 else 4, csb, 0,
                     rp.ctypes.data, col.ctypes.data, val.ctypes.data)
        o = cls._opts(devices, lane_width, accumulation, gather)
        h = C.c_void_p()
        _check(_lib().dg_multi_create(C.byref(view), C.byref(o), C.byref(h)), "dg_multi_create")
        return cls(h)

    @classmethod
    def generate(cls, profiles, devices: Sequence[int], *, gather: int = GATHER_PEER,
                 index_bytes: int = 0, lane_width: int = 32,
                 accumulation: int = ACCUM_EXACT) -> "MultiDoseEngine":
        arr, n = _profiles(profiles)
        o = cls._opts(devices, lane_width, accumulation, gather)
        h = C.c_void_p()
        _check(_lib().dg_multi_create_generated(arr, n, index_bytes, C.byref(o), C.byref(h)),
               "dg_multi_create_generated")
        return cls(h)

    def dose(self, x: np.ndarray, out: Optional[np.ndarray] = None) -> np.ndarray:
        """The full d on the host (each device downloads its slice)."""
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = _out_array(out, self.rows)
        _check(_lib().dg_multi_dose(self._h, x.ctypes.data, len(x), y.ctypes.data, 0),
               "dg_multi_dose")
        return y

    def dose_host_ptrs(self, x_ptr: int, x_len: int, y_ptr: int) -> None:
        _check(_lib().dg_multi_dose(self._h, C.c_void_p(x_ptr), x_len, C.c_void_p(y_ptr), 0),
               "dg_multi_dose")

    def dose_device(self, x_ptr: int, x_len: int) -> None:
        """x on devices[0]; d stays on the devices (device_d)."""
        _check(_lib().dg_multi_dose(self._h, C.c_void_p(x_ptr), x_len, None,
                                    X_ON_DEVICE | Y_ON_DEVICE), "dg_multi_dose")

    def device_d(self, i: int) -> tuple:
        """(full d, this shard's slice) device pointers on shard i's device."""
        f, s = C.c_void_p(), C.c_void_p()
        _check(_lib().dg_multi_device_d(self._h, i, C.byref(f), C.byref(s)), "dg_multi_device_d")
        return int(f.value), int(s.value)

    def shard(self, i: int) -> "DoseEngine":
        """Shard i as a (non-owning) DoseEngine view."""
        sh = C.c_void_p()
        _check(_lib().dg_multi_shard(self._h, i, C.byref(sh)), "dg_multi_shard")
        e = DoseEngine(sh)
        e._owner = False
        return e

    def last_timing(self) -> dict:
        t = _Timing()
        _check(_lib().dg_multi_last_timing(self._h, C.byref(t)), "dg_multi_last_timing")
        return {"ms_h2d": t.ms_h2d, "ms_kernels": t.ms_kernels, "ms_d2h": t.ms_d2h,
                "ms_total": t.ms_total}

    def close(self) -> None:
        if self._h:
            _lib().dg_multi_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


def _out_array(out: Optional[np.ndarray], n: int) -> np.ndarray:
    """A caller-supplied output array must be a writable, C-contiguous float64 array of n
    elements: the library writes n doubles through its pointer."""
    if out is None:
        return np.empty(n, dtype=np.float64)
    if not isinstance(out, np.ndarray) or out.dtype != np.float64 or out.size != n \
            or not out.flags.c_contiguous or not out.flags.writeable:
        raise ValueError(f"out must be a writable C-contiguous float64 array of {n} elements")
    return out


class PeerBuffer:
    """A device buffer of float64 that other processes can map (CUDA IPC, dg_ipc_*).

    ``PeerBuffer(n, device)`` allocates and exports (``handle``: 64 bytes to send to the peers);
    ``PeerBuffer.open(handle, n, device)`` maps a peer's buffer.  ``tensor()`` views it as a torch
    tensor through ``__cuda_array_interface__`` (no copy)."""

    def __init__(self, n: int, device: int = 0, *, _ptr: int = 0, _owner: bool = True,
                 _handle: bytes = b""):
        self.n, self.device, self.owner = int(n), int(device), _owner
        if _ptr:
            self.ptr, self.handle = _ptr, _handle
            return
        p = C.c_void_p()
        hbuf = C.create_string_buffer(64)
        _check(_lib().dg_ipc_alloc(self.n * 8, self.device, C.byref(p), hbuf), "dg_ipc_alloc")
        self.ptr, self.handle = int(p.value), hbuf.raw

    @classmethod
    def open(cls, handle: bytes, n: int, device: int = 0) -> "PeerBuffer":
        p = C.c_void_p()
        hbuf = C.create_string_buffer(bytes(handle), 64)
        _check(_lib().dg_ipc_open(hbuf, int(device), C.byref(p)), "dg_ipc_open")
        return cls(n, device, _ptr=int(p.value), _owner=False, _handle=bytes(handle))

    @property
    def __cuda_array_interface__(self):
        return {"shape": (self.n,), "typestr": "<f8", "data": (self.ptr, False), "version": 2,
                "strides": None}

    def tensor(self):
        import torch
        return torch.as_tensor(self, device=f"cuda:{self.device}")

    def close(self) -> None:
        if self.ptr:
            if self.owner:
                _lib().dg_ipc_free(C.c_void_p(self.ptr))
            else:
                _lib().dg_ipc_close(C.c_void_p(self.ptr))
            self.ptr = 0

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class ScatterEngine:
    """The column-scatter comparator (ddm::spmv_scatter_baseline, spmv.cpp:113-150) on the GPU:
    atomic-free, bit-identical to the reference for the same chunk_count."""

    def __init__(self, m: CsrMatrix, chunk_count: int = 1, *, device: int = -1):
        rp = np.ascontiguousarray(m.row_ptr, dtype=np.uint64)
        col = np.ascontiguousarray(m.col_indices, dtype=np.uint32)
        val = np.ascontiguousarray(m.values, dtype=_VDTYPE[m.precision])
        view = _View(m.rows, m.cols, m.nnz, m.precision, 2 if m.index_width == U16 else 4, 4, 0,
                     rp.ctypes.data, col.ctypes.data, val.ctypes.data)
        self._h = C.c_void_p()
        self.rows, self.cols = m.rows, m.cols
        _check(_lib().dg_scatter_create(C.byref(view), chunk_count, device, C.byref(self._h)),
               "dg_scatter_create")

    def dose(self, x: np.ndarray) -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.empty(self.rows, dtype=np.float64)
        _check(_lib().dg_scatter_dose(self._h, x.ctypes.data, len(x), y.ctypes.data, 0, None),
               "dg_scatter_dose")
        return y

    def dose_device(self, x_ptr: int, x_len: int, y_ptr: int, stream: int = 0) -> None:
        _check(_lib().dg_scatter_dose(self._h, C.c_void_p(x_ptr), x_len, C.c_void_p(y_ptr),
                                      X_ON_DEVICE | Y_ON_DEVICE | NO_SYNC,
                                      C.c_void_p(stream) if stream else None), "dg_scatter_dose")

    def close(self):
        if self._h:
            _lib().dg_scatter_destroy(self._h)
            self._h = None

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


def spmv_scatter_baseline(m: CsrMatrix, x: np.ndarray, chunk_count: int = 1, workers: int = 1,
                          *, device: int = -1) -> np.ndarray:
    """ddm::spmv_scatter_baseline semantics on the GPU (the CSC is built on the device)."""
    if len(x) != m.cols:
        raise Error(1 + Errc.DimensionMismatch, f"input vector length {len(x)} != {m.cols}")
    if chunk_count < 1 or workers < 1:
        raise Error(1 + Errc.InvalidConfig, "chunk_count and workers must be >= 1")
    with ScatterEngine(m, chunk_count, device=device) as e:
        return e.dose(x)


# ---------------------------------------------------------------- drop-in functions -------
def spmv_rowchunk(m: CsrMatrix, x: np.ndarray, cfg: RowChunkConfig = RowChunkConfig(),
                  *, device: int = -1) -> np.ndarray:
    """ddm::spmv_rowchunk on the GPU: bits equal the reference's for the same lane_width."""
    if cfg.workers < 1:
        raise Error(1 + Errc.InvalidConfig, "workers must be >= 1")
    if len(x) != m.cols:  # spmv.cpp:34-38: checked before the config, as the reference does
        raise Error(1 + Errc.DimensionMismatch,
                    f"input vector length {len(x)} != matrix columns {m.cols}")
    with DoseEngine.from_csr(m, lane_width=cfg.lane_width, device=device) as e:
        return e.dose(x)


def spmv_oracle(m: CsrMatrix, x: np.ndarray, *, device: int = -1) -> np.ndarray:
    """ddm::spmv_oracle semantics (sequential fp64 per row) == rowchunk with lane_width 1."""
    return spmv_rowchunk(m, x, RowChunkConfig(lane_width=1), device=device)


def checksum_bits(v: np.ndarray) -> int:
    v = np.ascontiguousarray(v, dtype=np.float64)
    out = C.c_uint64()
    _check(_lib().dg_checksum_bits(v.ctypes.data, len(v), 0, C.byref(out)), "dg_checksum_bits")
    return int(out.value)


def checksum_bits_device(ptr: int, n: int) -> int:
    out = C.c_uint64()
    _check(_lib().dg_checksum_bits(C.c_void_p(ptr), n, 1, C.byref(out)), "dg_checksum_bits")
    return int(out.value)


def traffic_bytes(rows: int, cols: int, nnz: int, value_bytes: int = 2, index_bytes: int = 2) -> int:
    return int(_lib().dg_traffic_bytes(rows, cols, nnz, value_bytes, index_bytes))


def partition_rows(row_ptr: np.ndarray, parts: int, bytes_per_nnz: int = 4) -> np.ndarray:
    rp = np.ascontiguousarray(row_ptr, dtype=np.uint64)
    b = np.empty(parts + 1, dtype=np.uint64)
    _check(_lib().dg_partition_rows(rp.ctypes.data, len(rp) - 1, bytes_per_nnz, parts,
                                    b.ctypes.data), "dg_partition_rows")
    return b


def partition_lengths(lengths: np.ndarray, parts: int, bytes_per_nnz: int = 4) -> np.ndarray:
    ln = np.ascontiguousarray(lengths, dtype=np.uint32)
    b = np.empty(parts + 1, dtype=np.uint64)
    _check(_lib().dg_partition_lengths(ln.ctypes.data, len(ln), bytes_per_nnz, parts,
                                       b.ctypes.data), "dg_partition_lengths")
    return b


def seeded_vector(n: int, seed: int) -> np.ndarray:
    """ddm::seeded_vector (bench.cpp:31-36): the reference benchmark's x."""
    out = np.empty(n, dtype=np.float64)
    _lib().dg_seeded_vector(n, seed, out.ctypes.data)
    return out


def generated_row_lengths(profiles, row_begin: int, row_end: int, device: int = -1) -> np.ndarray:
    arr, n = _profiles(profiles)
    out = np.empty(row_end - row_begin, dtype=np.uint32)
    _check(_lib().dg_generated_row_lengths(arr, n, row_begin, row_end, device, out.ctypes.data),
           "dg_generated_row_lengths")
    return out


def exported_symbols() -> Sequence[str]:
    return list(_SIGS)
