#!/bin/bash
# Round-2 ncu set, part 2: the CholeskyQR basis and the orthonormalisation core (cfg4), and the
# int8 first shrink + mode-0 norms of cfg5 (traffic for bench.py's roofline).
out=gpurun_out/r02
mkdir -p $out
B="python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^(cholqr_kernel|orth_core_kernel)$" -c 4 -o $out/orth_cfg4 $B --config cfg4 > $out/ncu_orth.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"^(ttm_i8_kernel|sqnorm_contig_kernel)$" -c 2 -o $out/stream_cfg5 $B --config cfg5 > $out/ncu_stream5.log 2>&1
ls -la $out/*.ncu-rep
