"""MXFP8 (1x32 blocks, E8M0 scales, E4M3 payload) — CPU oracle, TEST INFRASTRUCTURE ONLY.

Restates the reference's MXFP8 emulation (pkg/src/moelab):
  * e8m0_scale            formats.py:129-139  scale = 2^ceil(log2(amax / 448)), exponent
                                              clamped to [-127, 127]; amax == 0 -> 2^-127
  * quantize (MXFP8)      quant.py:166-201    1x32 blocks along the row (make_recipe
                                              quant.py:62-64: act_block = weight_block =
                                              (1, 32)); codes = E4M3.encode(x / scale)
  * E4M3 encode           formats.py:16-62    round-to-nearest-even on the value lattice
                                              (subnormals included), saturating at 448,
                                              sign in bit 7 (OCP layout)
  * dequantize-then-multiply is the reference's only GEMM path (quant.py:1-7).
Pinned by tests/test_mxfp8.py against codes and scales produced by the reference itself
(tests/golden/make_mxfp8_golden.py -> mxfp8_golden.npz).
"""
from __future__ import annotations

import numpy as np

E4M3_MAX = 448.0


def _e4m3_lattice():
    vals, codes = [0.0], [0]
    for e in range(16):
        for m in range(8):
            if e == 0:
                if m == 0:
                    continue
                v = (m / 8) * 2.0 ** (1 - 7)
            else:
                if e == 15 and m == 7:
                    continue  # NaN slot
                v = (1 + m / 8) * 2.0 ** (e - 7)
            vals.append(v)
            codes.append((e << 3) | m)
    order = np.argsort(vals)
    return np.array(vals)[order], np.array(codes)[order]


_VALS, _CODES = _e4m3_lattice()


def e4m3_encode(x: np.ndarray) -> np.ndarray:
    x = np.asarray(x, dtype=np.float64)
    mag = np.minimum(np.abs(x), E4M3_MAX)
    hi = np.clip(np.searchsorted(_VALS, mag, side="left"), 0, len(_VALS) - 1)
    lo = np.clip(hi - 1, 0, len(_VALS) - 1)
    lo = np.where(_VALS[hi] == mag, hi, lo)
    span = _VALS[hi] - _VALS[lo]
    with np.errstate(invalid="ignore", divide="ignore"):
        frac = np.where(span > 0, (mag - _VALS[lo]) / np.where(span > 0, span, 1.0), 0.0)
    take_hi = np.where(frac == 0.5, (_CODES[hi] & 1) == 0, frac > 0.5)
    codes = _CODES[np.where(take_hi, hi, lo)]
    return np.where(np.signbit(x), codes + 128, codes).astype(np.uint8)


def e4m3_decode(codes: np.ndarray) -> np.ndarray:
    codes = np.asarray(codes, dtype=np.int64)
    lut = np.full(128, np.nan)
    lut[_CODES] = _VALS
    v = lut[codes & 127]
    return np.where(codes >= 128, -v, v)


def e8m0_exponent(amax: np.ndarray) -> np.ndarray:
    amax = np.asarray(amax, dtype=np.float64)
    with np.errstate(divide="ignore"):
        e = np.ceil(np.log2(np.where(amax > 0, amax, 1.0) / E4M3_MAX))
    e = np.where(amax > 0, e, -127)
    return np.clip(e, -127, 127).astype(np.int64)


def quantize_mxfp8(x: np.ndarray):
    """x [rows, K] (K % 32 == 0) -> (codes uint8 [rows, K], scale codes uint8 [rows, K/32]
    with scale = 2^(code - 127))."""
    x = np.asarray(x, dtype=np.float64)
    r, k = x.shape
    blocks = x.reshape(r, k // 32, 32)
    e = e8m0_exponent(np.abs(blocks).max(axis=2))
    scaled = blocks / (2.0 ** e)[:, :, None]
    codes = e4m3_encode(scaled).reshape(r, k)
    return codes, (e + 127).astype(np.uint8)


def dequantize_mxfp8(codes: np.ndarray, scales: np.ndarray) -> np.ndarray:
    r, k = codes.shape
    v = e4m3_decode(codes).reshape(r, k // 32, 32)
    return (v * (2.0 ** (scales.astype(np.int64) - 127))[:, :, None]).reshape(r, k)


def tile_scales(scales: np.ndarray, rows_pad: int) -> np.ndarray:
    """Plain [rows, K/32] scale codes -> the GEMM's tiled layout: per (128-row tile, 128-wide K
    stage) a 512-byte chunk whose byte i*16 + c*4 + j is the scale of row tile*128 + c*32 + i,
    K-block stage*4 + j (the tcgen05.cp 32x128b.warpx4 source layout). Rows past `rows`
    are zero."""
    r, kb = scales.shape
    sp = np.zeros((rows_pad, kb), dtype=np.uint8)
    sp[:r] = scales
    t = sp.reshape(rows_pad // 128, 4, 32, kb // 4, 4)      # tile, c, i, stage, j
    return np.ascontiguousarray(t.transpose(0, 3, 2, 1, 4)).reshape(-1)
