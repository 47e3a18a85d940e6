"""Device time of fiber_compact_hits on one C2 launch's records (2^20 pairs, fiber A, D = 9):
50 calls queued behind a sleep kernel, so the host's enqueueing is not timed."""
import sys, torch
sys.path.insert(0, "/root/repo")
import paper_1811_03374_b200 as fx
from workloads import gen
w = gen.config2("A", n_rays=1 << 20, depth=22)
r, s, p = fx.to_device(w)
h = fx.intersect(r, s, p, 9)
n = h.shape[0]
out = torch.empty_like(h); idx = torch.empty(n, dtype=torch.int32, device="cuda"); cnt = torch.empty(1, dtype=torch.int32, device="cuda")
for _ in range(5): fx.compact_hits(h, out=out, idx=idx, count=cnt)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda._sleep(20_000_000)  # ~10 ms of GPU time: the host enqueues all 50 calls meanwhile
e0.record()
for _ in range(50): fx.compact_hits(h, out=out, idx=idx, count=cnt)
e1.record(); torch.cuda.synchronize()
print(f"compact 1M records: {e0.elapsed_time(e1)/50*1e3:.1f} us per call, hits {int(cnt.item())}")
