"""PCIe host<->device copy microbenchmark (diagnostics): 16 GiB pinned <-> device,
one copy vs chunks on several streams, each direction alone and both at once."""
import time
import torch

N = 16 << 30
dev = torch.empty(N // 2, dtype=torch.float16, device="cuda")
dev2 = torch.empty(N // 2, dtype=torch.float16, device="cuda")
h_in = torch.empty(N // 2, dtype=torch.float16).pin_memory()
h_out = torch.empty(N // 2, dtype=torch.float16).pin_memory()
streams = [torch.cuda.Stream() for _ in range(8)]


def run(h2d_chunks, d2h_chunks):
    torch.cuda.synchronize()
    t = time.perf_counter()
    for k, (src, dst, chunks, off) in enumerate([(h_in, dev, h2d_chunks, 0), (dev2, h_out, d2h_chunks, 4)]):
        if chunks == 0:
            continue
        n = src.numel()
        for c in range(chunks):
            s = streams[(off + c) % 8]
            lo, hi = c * n // chunks, (c + 1) * n // chunks
            with torch.cuda.stream(s):
                dst[lo:hi].copy_(src[lo:hi], non_blocking=True)
    torch.cuda.synchronize()
    return time.perf_counter() - t


for h, d in ((1, 0), (4, 0), (0, 1), (0, 4), (1, 1), (2, 2), (4, 4)):
    run(h, d)
    ts = min(run(h, d) for _ in range(3))
    moved = (N if h else 0) + (N if d else 0)
    print(f"H2D chunks {h}  D2H chunks {d}: {ts * 1e3:.1f} ms  {moved / ts / 1e9:.1f} GB/s", flush=True)
