"""Host<->device copy bandwidth with pinned memory (H2D, D2H, both at once),
one GPU or several at once: the bound on bench.py's e2e figure.
    python tools/pcie_probe.py                      # one GPU
    for i in 0 1 2 3; do LOCAL_RANK=$i python tools/pcie_probe.py & done; wait"""
import torch, time, os, sys
dev = int(os.environ.get("LOCAL_RANK", 0)); torch.cuda.set_device(dev)
N = 1 << 30
h = torch.empty(N, dtype=torch.uint8, pin_memory=True)
d = torch.empty(N, dtype=torch.uint8, device="cuda")
h2 = torch.empty(N, dtype=torch.uint8, pin_memory=True)
for name, fn in (("H2D", lambda: d.copy_(h, non_blocking=True)), ("D2H", lambda: h.copy_(d, non_blocking=True)),
                 ("both", None)):
    s2 = torch.cuda.Stream()
    for _ in range(2):
        torch.cuda.synchronize(); t = time.perf_counter()
        if fn: fn()
        else:
            d.copy_(h, non_blocking=True)
            with torch.cuda.stream(s2): h2[: N // 4].copy_(d[: N // 4], non_blocking=True)
        torch.cuda.synchronize(); dt = time.perf_counter() - t
    print(f"rank {dev} {name}: {N/dt/1e9:.1f} GB/s ({dt*1e3:.1f} ms)", flush=True)
