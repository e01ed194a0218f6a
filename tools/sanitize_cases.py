"""Small invocations of every kernel family, for compute-sanitizer (memcheck / racecheck /
synccheck) runs on the GPU box."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2603_08661_b200 as igs
from paper_2603_08661_b200 import sharded
from paper_2603_08661_b200.synth import random_cloud, synth_view

# 20 views: the 16-slot candidate / survivor ring wraps (views 16..19 reuse slots 0..3)
views = np.stack([synth_view(70, 150, 7000 + k) for k in range(20)])
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
# the sharded densify step at world 1 (keys / boundary / finalize / list-mode split / child index)
scene_s = igs.Scene3(pos, ls, q, o, sh, capacity=2 * n)
print(sharded.densify_step_sharded(scene_s, st2, cfg, 2000))
# fused 2-D split through densify_step, a fused split that must not write (budget), scene IO
m = 500
sc2 = igs.Scene2(np.random.default_rng(6).normal(size=(m, 2)), np.zeros((m, 2)), np.zeros(m),
                 np.zeros(m), np.ones((m, 3)), capacity=m + 100)
st3 = igs.DensifyStats(m)
igs.accumulate_grads(st3, np.random.default_rng(7).exponential(3e-4, m))
st3.set_edge_score(np.random.default_rng(8).random(m))
print(igs.densify_step(sc2, st3, igs.DensifyConfig(budget=m + 100), 2000))
small = igs.Scene3(pos[:64], ls[:64], q[:64], o[:64], sh[:64], capacity=70)
try:
    igs.las_split_batch(small, np.ones(64, bool))
except igs.BudgetError:
    pass
# large enough for the warp-per-tile LAS pre-pass (> 2 tiles per CTA) in both apply modes,
# and a sharded select whose length is not a multiple of 4 (the compact pass's row tails)
nb = 700_001
posb, lsb, qb, ob, shb = random_cloud(nb, 4, seed=9)
big = igs.Scene3(posb, lsb, qb, ob, shb, capacity=nb + nb // 10)
mb = np.random.default_rng(10).random(nb) < 0.05
igs.las_split_batch(big, mb)
from paper_2603_08661_b200 import las_split as LS
big2 = igs.Scene3(posb, lsb, qb, ob, shb, capacity=nb + nb // 10)
s2 = LS.split_async(big2, torch.from_numpy(mb).cuda(), igs.SplitConstants(), sparse=True)
LS.finish_split(big2, *(int(v) for v in s2.cpu()))
st4 = igs.DensifyStats(3001)
st4._grad_sum.copy_(torch.from_numpy(np.random.default_rng(11).exponential(3e-4, 3001)))
st4._accum_count = 1
st4.set_edge_score(np.random.default_rng(12).random(3001))
print(int(sharded.select_candidates_sharded(st4, cfg, 2000, 3001, 3001).sum()))
import tempfile
with tempfile.TemporaryDirectory() as d:
    igs.write_scene(scene, os.path.join(d, "s.igsp"))
    back = igs.read_scene(os.path.join(d, "s.igsp"), capacity=scene.count + 10)
    print(back.count)
torch.cuda.synchronize()
print("sanitize cases ok")
