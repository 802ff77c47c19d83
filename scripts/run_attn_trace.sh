touch paper_2605_29727_b200/csrc/attention.cu
BST_TRACE=1 python -c "from paper_2605_29727_b200.build import build; build()"
for a in "$@"; do echo "== $a"; timeout 120 python scripts/attn_trace_kt.py $a; done > gpurun_out/kt_trace.log 2>&1
cat gpurun_out/kt_trace.log
