"""Achievable HBM bandwidth for the fused pass's access pattern (2 streams read, 1 written,
equal sizes) vs plain copy (1 read, 1 written), measured with torch elementwise kernels and
CUDA events (best of 20).  Calibration only: the roofline peak stays MEASURED_PEAKS.json."""
import json
import torch

torch.cuda.set_device(0)
out = {}
for gib in (1, 2):
    n = gib * (1 << 30) // 4
    a = torch.rand(n, device="cuda")
    b = torch.rand(n, device="cuda")
    c = torch.empty_like(a)
    def t(fn, nbytes, reps=20):
        for _ in range(3):
            fn()
        best = 1e9
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); fn(); e1.record(); torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1) / 1e3)
        return nbytes / best / 1e9
    out[f"copy_{gib}GiB_GBs"] = t(lambda: c.copy_(a), 8 * n)
    out[f"add_2r1w_{gib}GiB_GBs"] = t(lambda: torch.add(a, b, out=c), 12 * n)
    out[f"axpby_2r1w_{gib}GiB_GBs"] = t(lambda: torch.add(a, b, alpha=0.5, out=c), 12 * n)
    del a, b, c
print(json.dumps(out))
