"""Raw PCIe copy rates on this box (pinned host buffers, one stream per
direction), to put the e2e leg's host<->device rate in context."""
import time

import torch

n_d2h, n_h2d = 5_376_000_000, 2_240_000_000
dev_o = torch.empty(n_d2h, dtype=torch.uint8, device="cuda")
dev_i = torch.empty(n_h2d, dtype=torch.uint8, device="cuda")
host_o = torch.empty(n_d2h, dtype=torch.uint8).pin_memory()
host_i = torch.empty(n_h2d, dtype=torch.uint8).pin_memory()
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for _ in range(2):
    host_o.copy_(dev_o, non_blocking=True)
    dev_i.copy_(host_i, non_blocking=True)
torch.cuda.synchronize()
for label, do_d2h, do_h2d in (("d2h", 1, 0), ("h2d", 0, 1), ("both", 1, 1)):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        if do_d2h:
            with torch.cuda.stream(s1):
                host_o.copy_(dev_o, non_blocking=True)
        if do_h2d:
            with torch.cuda.stream(s2):
                dev_i.copy_(host_i, non_blocking=True)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 3
    print(f"{label}: {dt * 1e3:.1f} ms  d2h {do_d2h * n_d2h / dt / 1e9:.1f} GB/s  "
          f"h2d {do_h2d * n_h2d / dt / 1e9:.1f} GB/s", flush=True)
