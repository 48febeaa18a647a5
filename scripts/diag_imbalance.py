"""Warp load imbalance of the streaming evaluator (GPU box, diagnostics
build: SQV_NVCC_EXTRA=-DSQV_DIAG_IMBAL, loaded with SQV_LIB): per CTA work
item, the longest of its 4 warps' item sequences against their mean.
usage: SQV_LIB=variants/imbal/libsqv.so python scripts/diag_imbalance.py [n_prims]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_17361_b200 as P  # noqa: E402
from paper_2511_17361_b200 import _lib  # noqa: E402
from paper_2511_17361_b200.scenegen import gen_frames  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
vox = P.Voxelizer(P.VoxelGridSpec(), P.VoxelizeConfig(), 18)
b = vox.to_device(gen_frames(20251117, 100, N, 18))
st = torch.zeros(4, dtype=torch.int64, device="cuda")
_lib.stats_attach(st)
vox(b)
torch.cuda.synchronize()
_lib.stats_attach(None)
mufu, pairs, mx, sm = (int(v) for v in st.cpu().tolist())
print({"n_prims": N, "sum_max": mx, "sum_items": sm, "imbalance_max_over_mean": 4 * mx / max(sm, 1)})
