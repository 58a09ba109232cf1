"""HBM bandwidth by traffic mix on this B200 (context for the tile kernel's write-heavy roofline):
write-only (fill), read-only (sum), copy (1:1), and a 1:3 read:write mix like C5's DRAM traffic (ncu: 4.0 GB read,
11.5 GB written per step).  CUDA events, best of 10, 4 GiB buffers (far above L2)."""
import json
import torch

def timed(fn, reps=10):
    best = 1e30
    for _ in range(3):
        fn()
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); a.record(); fn(); b.record(); torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) * 1e-3)
    return best

n = (4 << 30) // 8
x = torch.empty(n, dtype=torch.float64, device="cuda")
y = torch.empty(n, dtype=torch.float64, device="cuda")
x.fill_(1.0)
out = {}
t = timed(lambda: y.fill_(2.0)); out["write_only_GBs"] = n * 8 / t / 1e9
t = timed(lambda: x.sum()); out["read_only_GBs"] = n * 8 / t / 1e9
t = timed(lambda: y.copy_(x)); out["copy_1to1_GBs"] = 2 * n * 8 / t / 1e9
# 1:3 read:write: read a quarter-size slice once, write three full-size-quarter outputs
q = n // 4
xs = x[:q]
outs = [y[i * q:(i + 1) * q] for i in range(3)]
def mix():
    for o in outs:
        torch.mul(xs, 2.0, out=o) if o is outs[0] else o.fill_(3.0)
t = timed(mix); out["mix_1r_3w_GBs"] = (q * 8 * 4) / t / 1e9
out["device"] = torch.cuda.get_device_name()
print(json.dumps(out))
