import os, sys, time
sys.path.insert(0, os.getcwd())
import torch
import paper_2603_08661_b200 as igs
from paper_2603_08661_b200 import sharded, _lib
from paper_2603_08661_b200.schedule import is_warmup_step
n = 6_000_000
dev = torch.device("cuda", 0)
st = igs.DensifyStats(n, device=dev)
st._grad_sum.fill_(1.0); st._accum_count = 1; st.edge_score = torch.rand(n, dtype=torch.float64)
cfg = igs.DensifyConfig(budget=2 * n)
ops = sharded.CudaShardOps(n, dev)
L = ops.L
def T(label, f, reps=50):
    f(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t = time.perf_counter_ns(); f(); ts.append(time.perf_counter_ns() - t)
    ts.sort(); print(f"{label:40s} median {ts[len(ts)//2]/1e3:7.2f} us  min {ts[0]/1e3:7.2f}")
T("grad_sum.data_ptr", lambda: st._grad_sum.data_ptr())
T("edge_score.data_ptr", lambda: st.edge_score.data_ptr())
T("is_warmup_step", lambda: is_warmup_step(cfg, 2000))
T("stream_handle", lambda: _lib.stream_handle())
g, e = st._grad_sum.data_ptr(), st.edge_score.data_ptr()
h, w, wn, s = ops.hist.data_ptr(), ops.ws.data_ptr(), ops.ws.numel(), _lib.stream_handle()
T("igs_shard_keys C call only", lambda: L.igs_shard_keys(g, 1, e, n, 0.0002, 0, 0, h, w, wn, s))
T("ops.keys", lambda: ops.keys(st, cfg, 2000))
T("torch.empty(2,n)", lambda: torch.empty(2, n, dtype=torch.float64, device=dev))
T("stats.reset", lambda: st.reset(n))
T("cudaMemsetAsync via torch zero_ small", lambda: ops.hist.zero_())
T("igs_stream_synchronize", lambda: L.igs_stream_synchronize(s))
