"""HBM write / read / copy bandwidth of plain torch ops on a cfg2-sized buffer (development tool)."""
import torch
dev = torch.device("cuda")
o = torch.empty((65536, 6624), dtype=torch.float64, device=dev)
src = torch.empty_like(o)


def t(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


b = o.numel() * 8
for name, fn, mult in [("zero_", lambda: o.zero_(), 1), ("fill_", lambda: o.fill_(1.5), 1),
                       ("copy_", lambda: o.copy_(src), 2), ("sum", lambda: src.sum(), 1)]:
    ms = t(fn)
    print(f"{name}: {ms:.3f} ms {mult * b / ms / 1e6:.0f} GB/s")
