"""One large batched forward NTT launch group for ncu (C2 shape)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2407_07308_b200 as bc  # noqa: E402

ctx = bc.Context(bc.load_params("c2"))
x = torch.randint(0, 1 << 40, (128, ctx.n_cipher, ctx.n), dtype=torch.int64, device="cuda")
ws = ctx.workspace(128 * ctx.n_cipher * ctx.M * 8 + (64 << 20))
for _ in range(3):
    y = ctx.ntt_fwd(x, ws=ws)
torch.cuda.synchronize()
