"""TEST INFRASTRUCTURE ONLY -- ctypes front-end for the CPU checkers.

Two interchangeable back-ends with one Python surface:

* ``Oracle("port")``      -> oracle/liboracle.so, the plain-C restatement (ddm_oracle.c)
* ``Oracle("reference")`` -> oracle/_ref/libddmref.so, the reference library itself compiled
                             from /root/reference/proj/src (oracle/Makefile) + ref_shim.cpp

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline legs may import this module.
The product package (paper_2103_09683_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_LIB = os.path.join(HERE, "liboracle.so")
REF_LIB = os.path.join(HERE, "_ref", "libddmref.so")

HALF, SINGLE, DOUBLE = 0, 1, 2
U16, U32 = 0, 1
_VDTYPE = {HALF: np.uint16, SINGLE: np.float32, DOUBLE: np.float64}


class _Profile(C.Structure):
    _fields_ = [("rows", C.c_uint64), ("cols", C.c_uint64),
                ("target_nnz_ratio", C.c_double), ("empty_row_fraction", C.c_double),
                ("row_length_log_mean", C.c_double), ("row_length_log_sigma", C.c_double),
                ("locality_window", C.c_uint64), ("seed", C.c_uint64)]


class _Csr(C.Structure):
    _fields_ = [("rows", C.c_uint64), ("cols", C.c_uint64), ("nnz", C.c_uint64),
                ("precision", C.c_int32), ("index_width", C.c_int32),
                ("row_ptr", C.c_void_p), ("col", C.c_void_p), ("values", C.c_void_p)]


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

    def c(self) -> _Profile:
        return _Profile(self.rows, self.cols, self.target_nnz_ratio, self.empty_row_fraction,
                        self.row_length_log_mean, self.row_length_log_sigma,
                        self.locality_window, self.seed)


def liver_desk() -> Profile:  # matgen.cpp:13-27
    return Profile(29700, 6800, 0.0073, 0.70, 4.7661, 0.8278, 4096, 1)


def prostate_desk() -> Profile:  # matgen.cpp:29-43
    return Profile(10300, 5090, 0.0181, 0.70, 4.8880, 1.3165, 4096, 2)


def c1_profile() -> Profile:
    return Profile(1_000_000, 4096, 0.01, 0.70, 4.5741, 0.8278, 4096, 1)


@dataclass
class Csr:
    """Host CSR in the reference's in-memory encoding (sparse.hpp:93-108)."""
    rows: int
    cols: int
    precision: int
    index_width: int
    row_ptr: np.ndarray          # u64[rows+1]
    col: np.ndarray              # u32[nnz]
    values: np.ndarray           # u16 bits / f32 / f64 [nnz]
    _keep: list = field(default_factory=list, repr=False)

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1]) if len(self.row_ptr) else 0

    def c(self) -> _Csr:
        self.row_ptr = np.ascontiguousarray(self.row_ptr, dtype=np.uint64)
        self.col = np.ascontiguousarray(self.col, dtype=np.uint32)
        self.values = np.ascontiguousarray(self.values, dtype=_VDTYPE[self.precision])
        return _Csr(self.rows, self.cols, self.nnz, self.precision, self.index_width,
                    self.row_ptr.ctypes.data, self.col.ctypes.data, self.values.ctypes.data)

    def take_rows(self, rows: np.ndarray) -> "Csr":
        """Sub-matrix of the given rows (rows are independent in d = A.x, so the oracle on the
        sub-matrix is exact for those rows)."""
        rows = np.asarray(rows, dtype=np.int64)
        starts = self.row_ptr[rows].astype(np.int64)
        ends = self.row_ptr[rows + 1].astype(np.int64)
        lens = ends - starts
        rp = np.zeros(len(rows) + 1, dtype=np.uint64)
        np.cumsum(lens, out=rp[1:])
        idx = np.concatenate([np.arange(s, e) for s, e in zip(starts, ends)]) if len(rows) else \
            np.zeros(0, dtype=np.int64)
        return Csr(len(rows), self.cols, self.precision, self.index_width, rp,
                   self.col[idx], self.values[idx])


class OracleError(RuntimeError):
    def __init__(self, code: int, where: str):
        super().__init__(f"{where}: status {code}")
        self.code = code


class Oracle:
    def __init__(self, kind: str = "port"):
        self.kind = kind
        path = PORT_LIB if kind == "port" else REF_LIB
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle{' ref' if kind != 'port' else ''}`")
        self.lib = C.CDLL(path)
        p = "or_" if kind == "port" else "ref_"
        self._p = p
        L = self.lib
        P, D, U64 = C.c_void_p, C.c_double, C.c_uint64
        self._gen = getattr(L, p + "generate")
        self._gen.argtypes = [C.POINTER(_Profile), C.c_int, C.c_int, C.POINTER(_Csr)]
        self._free = getattr(L, p + "csr_free")
        self._free.argtypes = [C.POINTER(_Csr)]
        self._rowchunk = getattr(L, p + "spmv_rowchunk")
        self._rowchunk.argtypes = [C.POINTER(_Csr), P, U64, U64, U64, P]
        self._oracle = getattr(L, p + "spmv_oracle")
        self._oracle.argtypes = [C.POINTER(_Csr), P, U64, P]
        self._validate = getattr(L, p + "validate")
        self._validate.argtypes = [C.POINTER(_Csr)]
        self._checksum = getattr(L, p + "checksum_bits")
        self._checksum.argtypes = [P, U64]
        self._checksum.restype = U64
        self._decode = getattr(L, p + "decode_half")
        self._decode.argtypes = [C.c_uint16]
        self._decode.restype = D
        self._encode = getattr(L, p + "encode_half")
        self._encode.argtypes = [D, C.POINTER(C.c_uint16)]
        self._seeded = getattr(L, p + "seeded_vector")
        self._seeded.argtypes = [U64, U64, P]
        if kind != "port":
            L.ref_write_ddm.argtypes = [C.POINTER(_Csr), C.c_char_p]
            L.ref_read_ddm.argtypes = [C.c_char_p, C.POINTER(_Csr)]
            self._bench = L.ref_run_bench
            self._bench.argtypes = [C.POINTER(_Csr), C.c_int, U64, U64, U64, U64, U64, P,
                                    C.POINTER(C.c_uint64)]

    # --- construction -------------------------------------------------------------------
    def generate(self, prof: Profile, precision: int = HALF, index_width: int = -1) -> Csr:
        out = _Csr()
        rc = self._gen(C.byref(prof.c()), precision, index_width, C.byref(out))
        if rc:
            raise OracleError(rc, "generate")
        try:
            n = out.nnz
            rp = np.ctypeslib.as_array((C.c_uint64 * (out.rows + 1)).from_address(out.row_ptr)).copy()
            col = np.ctypeslib.as_array((C.c_uint32 * max(n, 1)).from_address(out.col))[:n].copy()
            vt = {HALF: C.c_uint16, SINGLE: C.c_float, DOUBLE: C.c_double}[out.precision]
            val = np.ctypeslib.as_array((vt * max(n, 1)).from_address(out.values))[:n].copy()
            return Csr(out.rows, out.cols, out.precision, out.index_width, rp, col, val)
        finally:
            self._free(C.byref(out))

    # --- dose path ----------------------------------------------------------------------
    def spmv_rowchunk(self, m: Csr, x: np.ndarray, lane_width: int = 32, workers: int = 1) -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.zeros(m.rows, dtype=np.float64)
        cm = m.c()
        rc = self._rowchunk(C.byref(cm), x.ctypes.data, len(x), lane_width, workers, y.ctypes.data)
        if rc:
            raise OracleError(rc, "spmv_rowchunk")
        return y

    def spmv_oracle(self, m: Csr, x: np.ndarray) -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.zeros(m.rows, dtype=np.float64)
        cm = m.c()
        rc = self._oracle(C.byref(cm), x.ctypes.data, len(x), y.ctypes.data)
        if rc:
            raise OracleError(rc, "spmv_oracle")
        return y

    def validate(self, m: Csr) -> int:
        cm = m.c()
        return int(self._validate(C.byref(cm)))

    def checksum_bits(self, v: np.ndarray) -> int:
        v = np.ascontiguousarray(v, dtype=np.float64)
        return int(self._checksum(v.ctypes.data, len(v)))

    def decode_half(self, h: int) -> float:
        return float(self._decode(h))

    def encode_half(self, x: float) -> int:
        out = C.c_uint16()
        rc = self._encode(x, C.byref(out))
        if rc:
            raise OracleError(rc, "encode_half")
        return int(out.value)

    def seeded_vector(self, n: int, seed: int) -> np.ndarray:
        v = np.empty(n, dtype=np.float64)
        self._seeded(n, seed, v.ctypes.data)
        return v

    def spmv_scatter(self, m: Csr, x: np.ndarray, chunk_count: int = 1, workers: int = 1) -> np.ndarray:
        """ddm::spmv_scatter_baseline on csr_to_csc(m) (spmv.cpp:113-150); reference only."""
        f = self.lib.ref_spmv_scatter
        f.argtypes = [C.POINTER(_Csr), C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint64, C.c_void_p]
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.zeros(m.rows, dtype=np.float64)
        cm = m.c()
        rc = f(C.byref(cm), x.ctypes.data, len(x), chunk_count, workers, y.ctypes.data)
        if rc:
            raise OracleError(rc, "spmv_scatter")
        return y

    def write_ddm(self, m: Csr, path: str) -> None:
        """ddm::write_ddm (io.cpp:67-96); reference back-end only."""
        cm = m.c()
        rc = self.lib.ref_write_ddm(C.byref(cm), path.encode())
        if rc:
            raise OracleError(rc, "write_ddm")

    def read_ddm_status(self, path: str) -> int:
        """ddm::read_ddm (io.cpp:103-168): 0 or 1 + Errc of the failure."""
        out = _Csr()
        rc = self.lib.ref_read_ddm(path.encode(), C.byref(out))
        if rc == 0:
            self._free(C.byref(out))
        return int(rc)

    def run_bench(self, m: Csr, algorithm: int = 1, lane_width: int = 32, workers: int = 1,
                  reps: int = 3, warmup: int = 1, vector_seed: int = 42) -> dict:
        """ddm::run_bench (bench.cpp:38-103); reference back-end only."""
        if self.kind == "port":
            raise RuntimeError("run_bench needs the reference back-end")
        out = (C.c_double * 5)()
        ck = C.c_uint64()
        cm = m.c()
        rc = self._bench(C.byref(cm), algorithm, lane_width, workers, reps, warmup, vector_seed,
                         out, C.byref(ck))
        if rc:
            raise OracleError(rc, "run_bench")
        return {"mean_seconds": out[0], "min_seconds": out[1], "effective_gbps": out[2],
                "gflops": out[3], "operational_intensity": out[4], "checksum": int(ck.value)}


def traffic_bytes(rows: int, cols: int, nnz: int, value_bytes: int = 2, index_bytes: int = 2) -> int:
    """ddm::traffic(dims_of(m), layout_of(m)).total_bytes() (perf_model.cpp:41-54)."""
    return (value_bytes + index_bytes) * nnz + 16 * rows + 8 * cols


def have_reference() -> bool:
    return os.path.exists(REF_LIB)
