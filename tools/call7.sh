cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
for args in "" "--nosel" "--hit 0" "--hit 0 --nosel" "--reqs 2 --seq 16384" "--reqs 2 --seq 16384 --nosel" "--reqs 1 --seq 4096"; do
  echo "== $args"; timeout 300 python tools/micro_select.py $args 2>&1 | tail -1
done
T=600 bash tools/gpu_tests.sh tests/test_gpu_attention.py
tail -30 gpurun_out/test_gpu_attention.log
timeout 300 python tools/micro_attn.py --check 2>&1 | tail -2
KVS_ATTN=4 timeout 300 python tools/micro_attn.py --check 2>&1 | tail -2
timeout 300 python tools/micro_attn.py --frac 1.0 2>&1 | tail -1
