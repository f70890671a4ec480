#!/usr/bin/env python
"""Host->device copy bandwidth from pinned memory on this box, by chunk size (what the loader can hope for)."""
import json
import torch

out = {}
dev = torch.device("cuda", 0)
for mb in (1.18, 4, 16, 64, 256):
    n = int(mb * 1e6)
    src = torch.empty(n, dtype=torch.uint8).pin_memory()
    dst = torch.empty(n, dtype=torch.uint8, device=dev)
    reps = max(4, int(2e9 / n))
    dst.copy_(src, non_blocking=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        dst.copy_(src, non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    out[f"{mb}MB"] = round(n * reps / (e0.elapsed_time(e1) * 1e-3) / 1e9, 2)
print(json.dumps({"h2d_GB_per_s_by_chunk": out, "device": torch.cuda.get_device_name(0)}))
