#!/bin/bash
# Round-2 final measurement set (GPU box, repo root): per-config bench lines with the CPU port
# beside them, the strict-fp64 cfg4 line, cfg4 / cfg5 launch lists, and ncu --set full captures
# of the int8 contraction (cfg4) and the DMMA power kernels (cfg5 mode 0) -- each ncu command
# only after the same command ran clean without ncu.
out=gpurun_out/r02b
mkdir -p $out
for c in cfg4 cfg1 cfg2 cfg3 cfg5; do
  timeout 900 python bench.py --config $c > $out/bench_$c.log 2>&1
done
LMRA_TTM_I8=0 timeout 600 python bench.py --config cfg4 --no-cpu-baseline > $out/bench_cfg4_fp64.log 2>&1
B="python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline"
for c in cfg4 cfg5; do
  $B --config $c > /dev/null 2>&1 || echo "bench $c failed"
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launch_$c.csv $B --config $c > /dev/null 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^(norms3_seg_kernel|ttm_i8_kernel)$" -c 3 -o $out/stream_cfg4 $B --config cfg4 > $out/ncu_stream.log 2>&1
python tools/power_probe.py cfg5 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"ttm_kernel|gram_kernel" -c 2 -o $out/power_cfg5 python tools/power_probe.py cfg5 > $out/ncu_power.log 2>&1
ls -la $out
