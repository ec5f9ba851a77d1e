"""One alg4 run on a scaled cfg4 tensor (default 512^3) -- for ncu captures of norms3 / core TTM."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2303_11612_b200 as P
from paper_2303_11612_b200.configs import scaled, generate_device
N = int(sys.argv[1]) if len(sys.argv) > 1 else 512
ctx = P.Context(0, torch.cuda.current_stream().cuda_stream)
bc = scaled("cfg4", [N, N, N])
x = generate_device(bc, ctx=ctx)
t = P.DenseTensor.device(x, bc.dims)
for _ in range(2):
    P.run_raw(bc.alg, t, bc.cfg, ctx=ctx).free()
torch.cuda.synchronize()
print("ok", N)
