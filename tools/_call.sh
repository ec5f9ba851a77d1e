mkdir -p gpurun_out/s4
LMRA_TIMELINE=1 timeout 600 python bench.py --config cfg1 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/s4/tl8_cfg1.log 2>&1
for c in cfg1 cfg2 cfg3; do timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/s4/b12_$c.log 2>&1; done
