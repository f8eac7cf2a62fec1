cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
for args in "" "--nosel" "--hit 0" "--reqs 2 --seq 16384" "--reqs 1 --seq 4096" "--reqs 32" "--reqs 300 --seq 512"; do
  echo "== $args"; timeout 300 python tools/micro_select.py $args 2>&1 | tail -2
done
T=600 bash tools/gpu_tests.sh tests/test_gpu_attention.py tests/test_gpu_dhd.py tests/test_gpu_engine.py
timeout 300 python tools/micro_attn.py 2>&1 | tail -1
timeout 300 python tools/micro_attn.py --frac 1.0 2>&1 | tail -1
KVS_BENCH_DEBUG=1 timeout 600 python bench.py --steps 10 > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -1 gpurun_out/bench.err; cut -c1-300 gpurun_out/bench.json; python -c "import json; d=json.load(open('gpurun_out/bench.json')); print(d['kernels'], d['roofline']['achieved'], d['e2e'])"
timeout 600 python tools/step_trace.py --steps 2 2>&1 | grep "ms/step" | head -14
