"""Guess-window diagnostics: per view, was the median taken from the window candidates (no C
tasks), how many candidates / survivors (reads the ViewCtl blocks of the edge workspace)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2603_08661_b200 as igs  # noqa: E402
from paper_2603_08661_b200 import _lib  # noqa: E402
from paper_2603_08661_b200.synth import synth_views_torch  # noqa: E402

B = int(os.environ.get("VIEWS", "200"))
views = synth_views_torch(B, 822, 1237, seed=1000, device="cuda")
out = torch.empty((B, 822, 1237), dtype=torch.float64, device="cuda")
igs.importance_batch(views, out=out)
torch.cuda.synchronize()
ws = [v for k, v in _lib._ws.items() if k[2] == "edge"][0]
ctl = ws[256:256 + 128 * B].cpu().numpy().view(np.uint32).reshape(B, 32)
# ViewCtl words: tiles_done, binfound, collect_done, select_done, cnt1, cnt2, b1, b2, r1(2),
# r2(2), npos(2), denom(2), median(2), c_claim, a_claim, nsurv, tca, a_done, wcenter, ncand, tc
nsurv, tca, wc, ncand, tc = ctl[:, 20], ctl[:, 21], ctl[:, 23], ctl[:, 24], ctl[:, 25]
b1 = ctl[:, 6].astype(np.int32)
hit = tc == 0
print(f"hits {hit.sum()}/{B}; candidates/survivors mean {np.mean(ncand / np.maximum(nsurv, 1)):.3f}")
print("first 20: wc", (wc[:20].astype(np.int64) - 1).tolist())
print("b1       ", b1[:20].tolist())
print("ncand    ", ncand[:20].tolist())
print("nsurv    ", nsurv[:20].tolist())
