"""L2 re-read probe: DRAM bytes of the fc1 forward grouped GEMM (pair engine) for a
power-of-two hidden size (row stride 8 KB) and a padded one (8 KB + 128 B)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2603_07685_b200 import gemm  # noqa: E402

dev = torch.device("cuda", 0)
E, per, m = 8, 4096, 14336
for h in ((4096,) if len(sys.argv) > 1 else (4096, 4160)):
    rows = E * per
    be = (torch.arange(rows // 128, device=dev, dtype=torch.int32) // (per // 128))
    nmb = torch.tensor([rows // 128], dtype=torch.int32, device=dev)
    x = torch.randn((rows, h), device=dev).to(torch.bfloat16)
    w1 = (torch.randn((E, 2 * m, h), device=dev) * h ** -0.5).to(torch.bfloat16)
    for _ in range(3):
        gemm.fc1_fwd(x, w1, be, nmb, pair=True)
    torch.cuda.synchronize()
    print("h", h, flush=True)
    del x, w1
    torch.cuda.empty_cache()
