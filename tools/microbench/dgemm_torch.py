"""cuBLAS DGEMM throughput via torch (fp64 8192^3): burst (best of 10) and sustained (4 s loop)."""
import json
import time

import torch

n = 8192
a = torch.randn(n, n, dtype=torch.float64, device="cuda")
b = torch.randn(n, n, dtype=torch.float64, device="cuda")
for _ in range(3):
    c = a @ b
torch.cuda.synchronize()
best = 1e30
for _ in range(10):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    c = a @ b
    e.record()
    e.synchronize()
    best = min(best, s.elapsed_time(e))
burst = 2 * n**3 / best / 1e9
t0 = time.time()
cnt = 0
s = torch.cuda.Event(enable_timing=True)
e = torch.cuda.Event(enable_timing=True)
s.record()
while time.time() - t0 < 4.0:
    c = a @ b
    cnt += 1
    if cnt % 4 == 0:
        torch.cuda.synchronize()
e.record()
e.synchronize()
sus = 2 * n**3 * cnt / s.elapsed_time(e) / 1e9
# tall-skinny shapes of the hot path: (50 x 1000) @ (1000 x 1e6)
q = torch.randn(50, 1000, dtype=torch.float64, device="cuda")
x = torch.randn(1000, 1000 * 1000, dtype=torch.float64, device="cuda")
for _ in range(3):
    y = q @ x
torch.cuda.synchronize()
best2 = 1e30
for _ in range(5):
    s.record()
    y = q @ x
    e.record()
    e.synchronize()
    best2 = min(best2, s.elapsed_time(e))
print(json.dumps({"dgemm_8192_burst_tflops": round(burst, 2), "dgemm_8192_sustained_tflops": round(sus, 2),
                  "dgemm_50x1000x1e6_ms": round(best2, 3),
                  "dgemm_50x1000x1e6_tflops": round(2 * 50 * 1000 * 1e6 / best2 / 1e9, 2)}))
