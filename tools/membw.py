"""Calibrate streaming bandwidth on this GPU with torch ops: copy (1R+1W) and add (2R+1W)."""
import torch
for dt in (torch.float64, torch.float32):
    n = (1 << 30) // (8 if dt == torch.float64 else 4) * 1  # 1 GiB per tensor
    a = torch.rand(n, device="cuda", dtype=dt); b = torch.rand(n, device="cuda", dtype=dt); c = torch.empty_like(a)
    for name, fn, nbytes in (("copy", lambda: c.copy_(a), 2), ("add", lambda: torch.add(a, b, out=c), 3)):
        for _ in range(3): fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        best = 1e9
        for _ in range(10):
            e0.record(); fn(); e1.record(); torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        print(f"{dt} {name}: {nbytes * n * a.element_size() / (best * 1e-3) / 1e9:.1f} GB/s")
