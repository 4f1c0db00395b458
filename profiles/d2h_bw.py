"""D2H bandwidth into pinned host buffers of growing size (host-side limit check for the c5 corner)."""
import torch, time
src = torch.empty(int(6.4e9)//2, dtype=torch.int16, device="cuda")
for gb in (6.4, 25.6, 51.2):
    n = int(gb * 1e9) // 2
    t0 = time.time()
    dst = torch.empty(n, dtype=torch.int16).pin_memory()
    tp = time.time() - t0
    torch.cuda.synchronize()
    t0 = time.time()
    off = 0
    while off < n:
        m = min(src.numel(), n - off)
        dst[off:off + m].copy_(src[:m], non_blocking=True)
        off += m
    torch.cuda.synchronize()
    dt = time.time() - t0
    print(f"pinned {gb} GB: pin {tp:.1f}s, D2H {gb/dt:.1f} GB/s")
    del dst
