"""PCIe probe: pinned H2D bandwidth with 1 vs 2 concurrent streams (1.08 GB buffers)."""
import torch
n = 135 * 1024 * 1024  # doubles = 1.08 GB
h = [torch.empty(n, dtype=torch.float64).pin_memory() for _ in range(2)]
d = [torch.empty(n, dtype=torch.float64, device="cuda") for _ in range(2)]
s = [torch.cuda.Stream() for _ in range(2)]
for mode in ("one stream", "two streams", "d2h+h2d"):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for rep in range(3):
        if mode == "one stream":
            d[0].copy_(h[0], non_blocking=True); d[1].copy_(h[1], non_blocking=True)
        elif mode == "two streams":
            for k in range(2):
                with torch.cuda.stream(s[k]):
                    d[k].copy_(h[k], non_blocking=True)
        else:
            with torch.cuda.stream(s[0]):
                d[0].copy_(h[0], non_blocking=True)
            with torch.cuda.stream(s[1]):
                h[1].copy_(d[1], non_blocking=True)
    torch.cuda.synchronize()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    gb = 3 * 2 * n * 8 / 1e9
    print(mode, f"{gb / (ms / 1e3):.1f} GB/s aggregate" )
