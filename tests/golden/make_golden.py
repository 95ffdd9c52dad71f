"""Regenerate tests/golden/ from the REFERENCE itself (oracle/_ref/libddmref.so, compiled from
/root/reference/proj/src by `make -C oracle ref`).  Run in the build container:

    python tests/golden/make_golden.py

Every number written here is produced by the unmodified reference library (ddm::generate,
ddm::seeded_vector, ddm::spmv_oracle, ddm::spmv_rowchunk, ddm::checksum_bits); the repo's C
restatement is pinned against these files by tests/test_oracle.py and the CUDA path by
tests/test_parity_gpu.py.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.oracle import (DOUBLE, HALF, SINGLE, U32, Csr, Oracle, c1_profile,  # noqa: E402
                           liver_desk, prostate_desk)


def fnv(b: bytes) -> str:
    port = Oracle("port")
    import ctypes as C
    port.lib.or_fnv1a64.restype = C.c_uint64
    port.lib.or_fnv1a64.argtypes = [C.c_char_p, C.c_uint64, C.c_uint64]
    return f"{port.lib.or_fnv1a64(b, len(b), 14695981039346656037):016x}"


def main() -> None:
    ref = Oracle("reference")
    out = {"_source": "oracle/_ref/libddmref.so (reference compiled from /root/reference/proj)"}
    lanes = [1, 2, 4, 8, 16, 32, 64, 128, 256, 1024]
    for name, prof in [("liver-desk", liver_desk()), ("prostate-desk", prostate_desk()),
                       ("c1", c1_profile())]:
        m = ref.generate(prof)
        x = ref.seeded_vector(m.cols, 42)
        e = {"rows": m.rows, "cols": m.cols, "nnz": m.nnz, "index_width": m.index_width,
             "values_fnv": fnv(m.values.tobytes()), "col_fnv": fnv(m.col.tobytes()),
             "row_ptr_fnv": fnv(m.row_ptr.tobytes()),
             "x_fnv": f"{ref.checksum_bits(x):016x}"}
        yo = ref.spmv_oracle(m, x)
        e["oracle"] = f"{ref.checksum_bits(yo):016x}"
        e["max_abs"] = float(np.abs(yo).max())
        e["rowchunk"] = {}
        for L in (lanes if name != "c1" else [1, 32, 64]):
            y = ref.spmv_rowchunk(m, x, L, 8)
            e["rowchunk"][str(L)] = f"{ref.checksum_bits(y):016x}"
        if name != "c1":
            e["precision"] = {}
            for prec in (SINGLE, DOUBLE):
                mp = ref.generate(prof, prec)
                e["precision"][str(prec)] = {
                    "rowchunk32": f"{ref.checksum_bits(ref.spmv_rowchunk(mp, x, 32, 8)):016x}",
                    "oracle": f"{ref.checksum_bits(ref.spmv_oracle(mp, x)):016x}"}
            # acceptance criterion 5 (acceptance.cpp:148-175): seeds 11..14, x seed + 1000
            e["seeds"] = {}
            for seed in (11, 12, 13, 14):
                p2 = type(prof)(**{**prof.__dict__, "seed": seed})
                ms = ref.generate(p2)
                xs = ref.seeded_vector(ms.cols, seed + 1000)
                e["seeds"][str(seed)] = {
                    "nnz": ms.nnz,
                    "rowchunk32": f"{ref.checksum_bits(ref.spmv_rowchunk(ms, xs, 32, 3)):016x}",
                    "oracle": f"{ref.checksum_bits(ref.spmv_oracle(ms, xs)):016x}"}
        out[name] = e
        print(name, e["nnz"], e["oracle"], e["rowchunk"]["32"], flush=True)

    # half codec: decode of every pattern (NaNs excluded: payload bits are not part of the
    # contract) and encode of a seeded sweep, from the reference.
    dec = np.array([ref.decode_half(b) for b in range(65536)])
    finite = np.isfinite(dec) | np.isinf(dec)
    out["half_decode_fnv"] = fnv(dec[finite].tobytes())
    rng = np.random.default_rng(7)
    sweep = np.concatenate([rng.uniform(-70000, 70000, 2000), rng.uniform(-1e-3, 1e-3, 2000),
                            np.ldexp(rng.uniform(0.5, 1, 1000), rng.integers(-30, 17, 1000))])
    enc = np.array([ref.encode_half(float(v)) for v in sweep], dtype=np.uint16)
    np.savez_compressed(os.path.join(HERE, "half_sweep.npz"), x=sweep, bits=enc)

    # acceptance.cpp:177-200: integer-valued matrices, every engine bit-exact
    from oracle.oracle import Oracle as _O  # noqa: F401
    ints = {}
    for prec in (HALF, SINGLE, DOUBLE):
        r = np.random.default_rng(500 + prec)
        dense = (r.integers(0, 10, (300, 120)) == 0) * r.integers(1, 9, (300, 120))
        rows, cols = np.nonzero(dense)
        rp = np.zeros(301, dtype=np.uint64)
        np.cumsum(np.bincount(rows, minlength=300), out=rp[1:])
        vals = dense[rows, cols].astype(np.float64)
        if prec == HALF:
            vals = np.array([ref.encode_half(v) for v in vals], dtype=np.uint16)
        elif prec == SINGLE:
            vals = vals.astype(np.float32)
        m = Csr(300, 120, prec, U32, rp, cols.astype(np.uint32), vals)
        x = r.integers(0, 16, 120).astype(np.float64)
        y = ref.spmv_oracle(m, x)
        ints[str(prec)] = {"y": f"{ref.checksum_bits(y):016x}"}
        np.savez_compressed(os.path.join(HERE, f"integer_{prec}.npz"), row_ptr=rp,
                            col=cols.astype(np.uint32), values=vals, x=x, y=y)
    out["integer"] = ints
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
