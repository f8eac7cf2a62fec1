#!/bin/bash
# compute-sanitizer passes (memcheck, racecheck, synccheck) over the GPU test
# files that drive the mbarrier/TMEM/cp.async pipelines (A1, D1, D2, D3,
# scatter, gather).  Run under gpurun; logs land in gpurun_out/san_*.log and
# a one-line-per-run summary in gpurun_out/sanitize_summary.txt.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
FILES=${FILES:-"tests/test_gpu_attention.py tests/test_gpu_dhd.py tests/test_gpu_select_batched.py tests/test_gpu_decode_select.py tests/test_gpu_batch.py"}
TOOLS=${TOOLS:-"memcheck racecheck synccheck"}
: > gpurun_out/sanitize_summary.txt
for tool in $TOOLS; do
  for f in $FILES; do
    b=$(basename $f .py)
    log=gpurun_out/san_${tool}_${b}.log
    timeout ${T:-900} compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 50 \
        python -m pytest $f -q -x -m gpu -p no:cacheprovider > $log 2>&1
    r=$?
    echo "$tool $b exit=$r $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|passed|failed' $log | tail -2 | tr '\n' ' ')" \
        | tee -a gpurun_out/sanitize_summary.txt
  done
done
