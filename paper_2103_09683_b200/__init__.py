"""B200-native dose SpMV (d = A.x over a dose-deposition matrix in its native encoding).

The compute lives in ``libdosegpu.so`` (hand-written sm_100a CUDA behind the C ABI in
include/dosegpu.h); this package is the host-side mirror of the reference's dose API.
"""
from .dose import (ACCUM_EXACT, ACCUM_FP32, DOUBLE, GATHER_NCCL, GATHER_NONE, GATHER_PEER,
                   HALF, SINGLE, U16, U32, CsrMatrix, DoseEngine, Errc, Error, MultiDoseEngine,
                   PeerBuffer, Profile, RowChunkConfig, checksum_bits,
                   checksum_bits_device, exported_symbols, generated_row_lengths,
                   partition_lengths, partition_rows, seeded_vector, spmv_oracle, spmv_rowchunk,
                   traffic_bytes)
from . import profiles

__all__ = [
    "ACCUM_EXACT", "ACCUM_FP32", "DOUBLE", "GATHER_NCCL", "GATHER_NONE", "GATHER_PEER", "HALF",
    "SINGLE", "U16", "U32", "CsrMatrix", "DoseEngine", "Errc", "Error", "MultiDoseEngine",
    "PeerBuffer", "Profile", "RowChunkConfig", "checksum_bits",
    "checksum_bits_device", "exported_symbols", "generated_row_lengths", "partition_lengths",
    "partition_rows", "seeded_vector", "spmv_oracle", "spmv_rowchunk", "traffic_bytes", "profiles",
]
