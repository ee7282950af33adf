"""Calibrate pure-write and copy bandwidth on the device (torch fill_ / copy_), CUDA events."""
import torch
x = torch.empty(2 ** 31, dtype=torch.int64, device="cuda")   # 16 GiB
y = torch.empty(2 ** 30, dtype=torch.int64, device="cuda")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for name, fn, nb in (("fill 16 GiB (write only)", lambda: x.fill_(7), x.numel() * 8),
                     ("zero 16 GiB (write only)", lambda: x.zero_(), x.numel() * 8),
                     ("copy 8 GiB (read + write)", lambda: x[:y.numel()].copy_(y), 2 * y.numel() * 8),
                     ("sum 16 GiB (read only)", lambda: x.sum(), x.numel() * 8)):
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print(f"{name}: {nb / best / 1e9:.0f} GB/s ({best:.2f} ms)")
