import sys; sys.path.insert(0, '/root/repo')
import torch
from torch.profiler import profile, ProfilerActivity
from bench import make_inputs, shard
from paper_1805_06572_b200.initializers import init_from_masks_batch
from paper_1805_06572_b200.synth import CONFIGS
for c in (4, 3):
    cfg = CONFIGS[c]
    Y, _, _, _ = make_inputs(cfg, shard(cfg, 0, 1))
    yd = torch.from_numpy(Y).cuda()
    init_from_masks_batch(yd); torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        init_from_masks_batch(yd); torch.cuda.synchronize()
    for e in prof.events():
        if e.device_type == torch.autograd.DeviceType.CUDA:
            print(c, e.name[:60], round((e.time_range.end - e.time_range.start) / 1e3, 3), "ms")
