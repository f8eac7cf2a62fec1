#!/bin/bash
# ncu evidence for one bench step: launch list (all kernels of the timed step)
# and a full-set capture of the selective attention kernel.  Run under gpurun.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
ARGS=${ARGS:-"--steps 1 --warmup 1 --profile"}
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none \
   --csv --log-file gpurun_out/launches.csv python bench.py $ARGS > gpurun_out/prof_bench.json 2> gpurun_out/prof_bench.err
echo "launch list rc=$?"
if [ -n "$FULL" ]; then
  for k in $FULL; do
    timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on \
      -k regex:$k -c 1 -o gpurun_out/prof_$k python bench.py $ARGS > /dev/null 2> gpurun_out/prof_$k.err
    echo "full $k rc=$?"
  done
fi
