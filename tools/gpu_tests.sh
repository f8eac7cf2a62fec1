#!/bin/bash
# Run the GPU test files one by one under coreutils timeout (a hung kernel
# kills only its own process); logs land in gpurun_out/.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt
FILES=${@:-tests/test_gpu_*.py}
rc=0
for f in $FILES; do
  b=$(basename $f .py)
  timeout ${T:-420} python -m pytest $f -q -x -m gpu -p no:cacheprovider > gpurun_out/$b.log 2>&1
  r=$?
  echo "$b exit=$r $(tail -1 gpurun_out/$b.log)"
  [ $r -ne 0 ] && rc=1
done
if [ -n "$SMOKE" ]; then timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit=$? $(tail -1 gpurun_out/smoke.log)"; fi
exit $rc
