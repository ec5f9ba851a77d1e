#!/bin/bash
# times the cfg4-shaped TTMs under each LMRA_TTM_VARIANT (K chunk / stages)
for V in 0 1 2 3; do
  echo "variant $V"
  LMRA_TTM_VARIANT=$V timeout 300 python tools/bench_primitives.py 2>&1 | grep -E "w(15|30|50|60)_tflops"
done
