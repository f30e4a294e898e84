import sys, time
sys.path.insert(0, '.')
import torch
from paper_2507_09029_b200 import engine, masking, zoo
dev = torch.device('cuda', 0)
topo = zoo.resnet18_cifar_topology()
a = masking.build_assignment(topo, 'neuron', 8, 4, seed=1)
d = topo.total
reps = [torch.randn(d, device=dev) * a.param_masks[w] for w in range(8)]
check = a.uncovered_params > 0
def t(f, n=200):
    for _ in range(10): f()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n): f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e6
gbar = torch.empty(d, device=dev)
st = torch.zeros(1, dtype=torch.int32, device=dev)
print('aggregate call us', t(lambda: engine.aggregate(reps, a)))
print('_bind only us', t(lambda: engine._bind(reps, a, out=gbar, writeback=False, check_uncovered=check, status=st)))
prep = engine.PreparedSync(reps, a, writeback=False, out=gbar, check_uncovered=check, status=st)
print('prepared launch (async) us', t(prep.launch))
def ps():
    prep.launch(); st.item()
print('prepared launch + status item us', t(ps))
print('torch.empty + zeros us', t(lambda: (torch.empty(d, device=dev), torch.zeros(1, dtype=torch.int32, device=dev))))
