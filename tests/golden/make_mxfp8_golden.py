"""Golden MXFP8 codes / scales from the REFERENCE quantizer (pkg/src/moelab/quant.py:166-201,
formats.py:16-139).

Run in the build container (the only place /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_mxfp8_golden.py

Writes tests/golden/mxfp8_golden.npz: bf16-representable inputs (normal, tiny, huge, ties,
zeros, saturating blocks) with the reference's E4M3 codes and E8M0 scale codes.
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

REF_SRC = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent / "mxfp8_golden.npz"


def bf16_round(x):
    u = np.asarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) >> 16 << 16
    return u.astype(np.uint32).view(np.float32).astype(np.float64)


def main() -> None:
    sys.dont_write_bytecode = True
    sys.path.insert(0, str(REF_SRC))
    from moelab.quant import make_recipe, quantize  # noqa: E402 (reference)

    rng = np.random.default_rng(32)
    rows = []
    rows.append(rng.normal(size=(8, 256)))
    rows.append(rng.normal(size=(4, 256)) * 1e-3)
    rows.append(rng.normal(size=(4, 256)) * 3e4)
    z = np.zeros((2, 256))
    z[1, 40] = 1.0
    rows.append(z)
    # exact powers of two / ties relative to the block scale
    t = np.tile(np.array([448.0, 1.0, 1.0625, 1.1875, -0.0, 2.0 ** -9, 3 * 2.0 ** -10, 240.0]),
                (2, 32))
    rows.append(t)
    rows.append(rng.standard_t(2, size=(6, 256)) * 10)
    x = bf16_round(np.concatenate(rows, axis=0))
    q = quantize(x, make_recipe("mxfp8"), "activation")
    codes = q.codes.astype(np.int64)
    np.savez_compressed(OUT, x=x.astype(np.float32), codes=codes.astype(np.uint8),
                        scales=np.asarray(q.block_scale_codes, dtype=np.int64).astype(np.uint8),
                        dequant=q.dequantize())
    print(f"wrote {OUT}: {x.shape}")


if __name__ == "__main__":
    main()
