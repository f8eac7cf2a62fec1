cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 300 python tools/micro_select.py 2>&1 | tail -3
timeout 300 python tools/micro_select.py --reqs 32 2>&1 | tail -1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dhd_select_fused -s 2 -c 1 -o gpurun_out/prof_select python tools/micro_select.py --iters 2 > /dev/null 2>&1; echo ncu rc=$?
T=600 bash tools/gpu_tests.sh tests/test_gpu_engine.py tests/test_gpu_dhd.py
KVS_BENCH_DEBUG=1 timeout 600 python bench.py --steps 10 > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -1 gpurun_out/bench.err; cut -c1-400 gpurun_out/bench.json
