"""Named matrix profiles: the reference's desk profiles and the BASELINE.json configs C1-C5.

Desk profiles: /root/reference/proj/src/matgen.cpp:13-43.  C1-C5: SURVEY.md 8(d) (log-normal
log_mean solved as ln(ratio*cols/(1-empty)) - sigma^2/2).
"""
from __future__ import annotations

from .dose import Profile


def liver_desk() -> Profile:  # matgen.cpp:13-27
    return Profile(29700, 6800, 0.0073, 0.70, 4.7661, 0.8278, 4096, 1)


def prostate_desk() -> Profile:  # matgen.cpp:29-43
    return Profile(10300, 5090, 0.0181, 0.70, 4.8880, 1.3165, 4096, 2)


def c1() -> Profile:
    """1M voxels x 4,096 spots, ~1%: the oracle config (BASELINE.json configs[0])."""
    return Profile(1_000_000, 4096, 0.01, 0.70, 4.5741, 0.8278, 4096, 1)


def c2(rows: int = 8_000_000, seed: int = 2) -> Profile:
    """8M voxels x 40k spots, ~3.2e9 nnz, skewed (prostate sigma): BASELINE.json configs[1]."""
    return Profile(rows, 40_000, 0.01, 0.70, 6.3288, 1.3165, 4096, seed)


def c4_beams(rows: int = 2_970_000) -> list:
    """Six 32,768-spot beams (seeds 11..16), hstacked -> 196,608 columns, U32 indices."""
    return [Profile(rows, 32_768, 0.0073, 0.70, 6.3386, 0.8278, 4096, 11 + b) for b in range(6)]


def c5_scenarios(rows: int = 88_000_000) -> list:
    """Nine robust-planning scenarios (seeds 101..109), each 88M x 40k."""
    return [Profile(rows, 40_000, 0.01, 0.70, 6.3288, 1.3165, 4096, 101 + s) for s in range(9)]


NAMED = {"liver-desk": liver_desk, "prostate-desk": prostate_desk, "c1": c1, "c2": c2}
