"""Oracle: saturating bandwidth curve (C-12).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Paper, Sec. 7: "NVLink bandwidth is poor for small data
transfers, e.g. between two A100 GPUs, the copy bandwidth of a 4MB buffer is
50 GB/s and 64 MB buffer is 200 GB/s."  The curve shape is SPEC's
(S:50-66): B(s) = peak * s / (s + half), calibrated in closed form from two
points; here also fitted by least squares to a measured sweep (config C5).
"""
from __future__ import annotations

from typing import Sequence, Tuple


def effective_bandwidth(peak: float, half: float, s: float) -> float:
    """B(s) = peak * s / (s + half)."""
    if s <= 0:
        raise ValueError("size must be > 0")
    return peak * s / (s + half)


def calibrate(s1: float, b1: float, s2: float, b2: float) -> Tuple[float, float]:
    """Two-point closed form:
    half = s1*s2*(b2-b1) / (b1*s2 - b2*s1);  peak = b1*(s1+half)/s1."""
    den = b1 * s2 - b2 * s1
    if den <= 0 or b2 <= b1:
        raise ValueError("no saturating curve through these points")
    half = s1 * s2 * (b2 - b1) / den
    peak = b1 * (s1 + half) / s1
    return peak, half


def fit(sizes: Sequence[float], bws: Sequence[float]) -> Tuple[float, float]:
    """Least squares in the reciprocal domain: 1/B = 1/peak + (half/peak)/s,
    a straight line in x = 1/s.  Returns (peak, half)."""
    xs = [1.0 / s for s in sizes]
    ys = [1.0 / b for b in bws]
    n = len(xs)
    mx, my = sum(xs) / n, sum(ys) / n
    sxx = sum((x - mx) ** 2 for x in xs)
    sxy = sum((x - mx) * (y - my) for x, y in zip(xs, ys))
    slope = sxy / sxx
    icpt = my - slope * mx
    peak = 1.0 / icpt
    return peak, slope * peak


def transfer_time(peak: float, half: float, total: float, nbuf: int, lat: float = 0.0) -> float:
    """nbuf equal buffers: nbuf * (lat + (total/nbuf)/B(total/nbuf))."""
    s = total / nbuf
    return nbuf * (lat + s / effective_bandwidth(peak, half, s))
