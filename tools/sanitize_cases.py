"""Small invocations of every kernel family, for compute-sanitizer (memcheck / racecheck /
synccheck) runs on the GPU box."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2603_08661_b200 as igs
from paper_2603_08661_b200 import sharded
from paper_2603_08661_b200.synth import random_cloud, synth_view

views = np.stack([synth_view(70, 150, 7000 + k) for k in range(3)])
igs.importance_batch(torch.from_numpy(views).cuda())
igs.importance_batch(torch.from_numpy(views[:, :, :, 0].copy()).cuda(), median=False)
igs.importance_pipeline(views[0], nms=False)
igs.median_normalize(np.random.default_rng(0).random(5001))
imp = igs.importance_pipeline(views[0])
igs.sample_scores(imp, np.random.default_rng(1).uniform(-2, 150, (777, 2)))
n = 3000
pos, ls, q, o, sh = random_cloud(n, 16, seed=3)
scene = igs.Scene3(pos, ls, q, o, sh, capacity=2 * n)
st = igs.DensifyStats(n)
igs.accumulate_position_grads(st, np.random.default_rng(2).standard_normal((n, 2)) * 3e-4)
st.set_edge_score(np.random.default_rng(3).random(n))
cfg = igs.DensifyConfig(budget=2 * n, growth_cap=0.3)
print(igs.densify_step(scene, st, cfg, 2000))
st2 = igs.DensifyStats(n)
st2._grad_sum.copy_(torch.from_numpy(np.random.default_rng(4).exponential(3e-4, n)))
st2._accum_count = 1
st2.set_edge_score(np.random.default_rng(5).random(n))
print(int(sharded.select_candidates_sharded(st2, cfg, 2000, n, n).sum()))
torch.cuda.synchronize()
print("sanitize cases ok")
