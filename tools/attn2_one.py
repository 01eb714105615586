#!/usr/bin/env python
"""One C2-shaped launch of the CTA-pair attention (QVK_ATTN_2CTA=1) after a warm-up — the ncu target."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2505_16175_b200 as qp  # noqa: E402

os.environ["QVK_ATTN_2CTA"] = os.environ.get("QVK_ATTN_2CTA", "1")
dev = torch.device("cuda", 0)
sizes = [4096] * 16
q = torch.cat([qp.synth_bf16(1, 3, 0, i, n, 28, 128, False, dev) for i, n in enumerate(sizes)])
k = torch.cat([qp.synth_bf16(1, 1, 0, i, n, 4, 128, True, dev) for i, n in enumerate(sizes)])
v = torch.cat([qp.synth_bf16(1, 2, 0, i, n, 4, 128, False, dev) for i, n in enumerate(sizes)])
g = qp.GroupPlan.from_sizes(sizes, 0.5).to(dev)
for _ in range(3):
    qp.attention(q, k, v, g, 28, 4)
torch.cuda.synchronize()
