import time, torch, numpy as np, sys
sys.path.insert(0, '.')
from paper_2507_09029_b200 import masking, zoo, engine
dev = torch.device('cuda', 0)
topo = zoo.resnet18_cifar_topology(); d = topo.total
a = masking.build_assignment(topo, 'block', 8, 4, seed=1)
host = []
for w in range(8):
    t = torch.empty(d, pin_memory=True); t.normal_(); host.append(t.numpy())
h = torch.from_numpy(host[0]); print('from_numpy pinned:', h.is_pinned())
dst = [torch.empty(d, device=dev) for _ in range(8)]
def tm(f, n=5):
    f(); torch.cuda.synchronize(); t0=time.perf_counter()
    for _ in range(n): f()
    torch.cuda.synchronize(); return (time.perf_counter()-t0)/n*1e3
print('8 full H2D ms', tm(lambda: [dst[w].copy_(torch.from_numpy(host[w]), non_blocking=True) for w in range(8)]))
plan = a.sync_plan()
print('ranges per worker', [len(plan.worker_ranges(w)) for w in range(8)])
print('range H2D ms', tm(lambda: [dst[w][s:s+l].copy_(torch.from_numpy(host[w])[s:s+l], non_blocking=True) for w in range(8) for s,l in plan.worker_ranges(w)]))
out = torch.empty(d, pin_memory=True); g = torch.empty(d, device=dev)
print('D2H ms', tm(lambda: out.copy_(g, non_blocking=True)))
print('aggregate ms', tm(lambda: engine.aggregate(host, a)))
engine.HOST_CHUNKS = 1
print('aggregate 1 chunk ms', tm(lambda: engine.aggregate(host, a)))
engine.HOST_CHUNKS = 4
print('aggregate 4 chunk ms', tm(lambda: engine.aggregate(host, a)))
