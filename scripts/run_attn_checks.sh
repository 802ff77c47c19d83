timeout 300 python -m pytest tests/test_gpu_attention.py -x -q 2>&1 | tail -5 > gpurun_out/t_attn.log
timeout 300 python scripts/bench_attention.py 2048 32768 > gpurun_out/attn_bench_kt.log 2>&1
touch paper_2605_29727_b200/csrc/attention.cu
BST_TRACE=1 python -c "from paper_2605_29727_b200.build import build; build()"
for a in "2048 17" "32768 17" "32768 65"; do echo "== $a"; timeout 120 python scripts/attn_trace_kt.py $a; done > gpurun_out/kt_trace.log 2>&1
cat gpurun_out/t_attn.log gpurun_out/attn_bench_kt.log; head -12 gpurun_out/kt_trace.log
