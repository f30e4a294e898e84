import sys, torch
sys.path.insert(0, '/root/repo')
from paper_2507_09029_b200 import masking, train
dev = torch.device("cuda", 0)
gen = torch.Generator(device=dev); gen.manual_seed(0)
batches = [(torch.randn(64, 3, 32, 32, generator=gen, device=dev), torch.randint(0, 10, (64,), generator=gen, device=dev)) for _ in range(8)]
model = train.build_resnet18(dev)
a = masking.build_assignment(model.topology, "block", 8, 8, seed=1)
tr = train.SubnetTrainer(model, a, lr=0.02)
for _ in range(2): tr.step(batches)
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CPU, torch.profiler.ProfilerActivity.CUDA], record_shapes=True) as prof:
    tr.step(batches[:1] * 8); torch.cuda.synchronize()
t = prof.key_averages(group_by_input_shape=True).table(sort_by="cuda_time_total", row_limit=25)
print("\n".join(l[:60] + l[150:] for l in t.splitlines()))
