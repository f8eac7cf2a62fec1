cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
for args in "" "--nosel" "--hit 0" "--reqs 2 --seq 16384" "--reqs 1 --seq 4096" "--reqs 32" "--reqs 300 --seq 512" "--reqs 1 --seq 20000"; do
  echo "== $args"; timeout 300 python tools/micro_select.py $args 2>&1 | tail -2
done
T=600 bash tools/gpu_tests.sh tests/test_gpu_dhd.py tests/test_gpu_engine.py
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dhd_select_fused -s 2 -c 1 -o gpurun_out/prof_select3 python tools/micro_select.py --iters 2 > /dev/null 2>&1; echo ncu rc=$?
