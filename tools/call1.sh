cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
SMOKE=1 T=600 bash tools/gpu_tests.sh > gpurun_out/tests_summary.txt 2>&1; echo "tests rc=$?" >> gpurun_out/tests_summary.txt
cat gpurun_out/tests_summary.txt
timeout 600 python bench.py > gpurun_out/bench_fwd3.json 2> gpurun_out/bench_fwd3.err; echo "bench3 rc=$?"; tail -c 3000 gpurun_out/bench_fwd3.json
KVS_ATTN=4 timeout 600 python bench.py > gpurun_out/bench_fwd4.json 2> gpurun_out/bench_fwd4.err; echo "bench4 rc=$?"; tail -c 3000 gpurun_out/bench_fwd4.json
KVS_ATTN=4 timeout 600 python -m pytest tests/test_gpu_engine.py -q -x -m gpu -p no:cacheprovider 2>&1 | tail -3
