#!/bin/bash
# Round-2 ncu set (GPU box, repo root): launch lists (cfg4, cfg5) and --set full captures of the
# top kernels -- each command only after the same command ran clean without ncu.
out=gpurun_out/r02
mkdir -p $out
B="python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline"
for c in cfg4 cfg5; do
  $B --config $c > /dev/null 2>&1 || echo "bench $c failed"
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launch_$c.csv $B --config $c > /dev/null 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^(orth_core_kernel|cholqr_kernel|chunk_walk_kernel)$" -c 8 -o $out/latency_cfg4 $B --config cfg4 > $out/ncu_latency.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^(norms3_seg_kernel|ttm_i8_kernel|segment_total_kernel)$" -c 5 -o $out/stream_cfg4 $B --config cfg4 > $out/ncu_stream.log 2>&1
ls -la $out
