"""Same-box A/B: width-wise (C3) trainer step with the batched slice launches
(one extract + one write-back for all workers, models.SliceBatch) vs the
per-worker launches (2 x N).  Graphed steps, CUDA events, alternating."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2507_09029_b200 import masking, train  # noqa: E402


class PerWorker(train.SubnetTrainer):
    def _step_eager(self, batches, cache: bool = True):
        losses = [self._compact_step_bf16(w, x, y, cache) for w, (x, y) in enumerate(batches)]
        self._sync()
        return torch.stack(losses).mean()


def main():
    dev = torch.device("cuda", 0)
    gen = torch.Generator(device=dev)
    gen.manual_seed(0)
    batches = [(torch.randn(64, 3, 32, 32, generator=gen, device=dev),
                torch.randint(0, 10, (64,), generator=gen, device=dev)) for _ in range(8)]
    trs = {}
    for tag, cls in (("batched", train.SubnetTrainer), ("per_worker", PerWorker)):
        m = train.build_resnet18(dev)
        a = masking.build_assignment(m.topology, "neuron", 8, 4, seed=1)
        trs[tag] = cls(m, a, lr=0.02, sync_layout=True, graphed=True)
        for _ in range(3):
            trs[tag].step(batches)
    torch.cuda.synchronize()
    res = {k: [] for k in trs}
    for rep in range(6):
        for tag, tr in trs.items():
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            for _ in range(20):
                tr.step(batches)
            e.record()
            torch.cuda.synchronize()
            res[tag].append(s.elapsed_time(e) / 20)
    a_, b_ = (trs["batched"].theta(), trs["per_worker"].theta())
    print({k: round(sorted(v)[len(v) // 2], 3) for k, v in res.items()}, "theta equal:", bool(torch.equal(a_, b_)))


if __name__ == "__main__":
    main()
