"""Host link bandwidth of this box: pinned H2D / D2H of the bench's per-step
volumes (134 MB of layouts in, 25 MB of costs out), alone and concurrent."""
import torch

n_in, n_out = 134217728, 25165824
hi = torch.empty(n_in, dtype=torch.uint8).pin_memory()
ho = torch.empty(n_out, dtype=torch.uint8).pin_memory()
di = torch.empty(n_in, dtype=torch.uint8, device="cuda")
do = torch.empty(n_out, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for name, fn in (("H2D 134 MB", lambda: di.copy_(hi, non_blocking=True)),
                 ("D2H 25 MB", lambda: ho.copy_(do, non_blocking=True))):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        fn()
    b.record(); torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 10
    nb = n_in if name.startswith("H2D") else n_out
    print(f"{name}: {ms:.3f} ms, {nb / ms / 1e6:.1f} GB/s")
