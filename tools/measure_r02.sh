#!/bin/bash
# Round-2 measurement set (run on the GPU box from the repo root): per-config bench lines with the
# CPU port beside them, the reference arm per config, the strict-fp64 (LMRA_TTM_I8=0) cfg4 line,
# the cfg4 launch list, and ncu --set full captures of the top kernels.
out=gpurun_out/r02
mkdir -p $out
for c in cfg4 cfg1 cfg2 cfg3 cfg5; do
  timeout 900 python bench.py --config $c > $out/bench_$c.log 2>&1
done
LMRA_TTM_I8=0 timeout 600 python bench.py --config cfg4 --no-cpu-baseline > $out/bench_cfg4_fp64.log 2>&1
for c in cfg1 cfg2 cfg3 cfg5 cfg4; do
  timeout 1500 python bench.py --impl reference --config $c --steps 3 --warmup 1 > $out/ref_$c.log 2>&1
done
