"""One MXFP8 fc2 launch (CTA pair, 256-wide tiles) after a warm-up launch, for ncu."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2603_07685_b200 import gemm  # noqa: E402

dev = torch.device("cuda", 0)
E, per, h, m = 8, 4096, 4096, 14336
rows = E * per
be = (torch.arange(rows // 128, device=dev, dtype=torch.int32) // (per // 128))
nmb = torch.tensor([rows // 128], dtype=torch.int32, device=dev)
act = torch.randn((rows, m), device=dev).to(torch.bfloat16)
w2 = (torch.randn((E, h, m), device=dev) * m ** -0.5).to(torch.bfloat16)
aq, asf, _ = gemm.mxfp8_quantize(act)
w2q, w2sf = gemm.mxfp8_quantize_weight(w2)
for _ in range(2):
    gemm.mxfp8_gemm(aq, asf, w2q, w2sf, E, be, nmb, h, pair=True, wide=True)
torch.cuda.synchronize()
print("ok")
