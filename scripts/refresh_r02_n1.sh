#!/bin/bash
# Final 1-GPU bench lines for profiles/r02 (run under gpurun, 1 GPU).
set -u
O=gpurun_out/r02
mkdir -p $O
run1() { timeout 600 python bench.py "$@" 2>>$O/n1_err.log | tail -1; }
run1 > $O/bench_mixtral_n1.json
run1 --config configs/dsv3_layer.yaml --steps 5 --no-cpu-baseline > $O/bench_dsv3_n1.json
run1 --config configs/mixtral_layer_fp32.yaml --steps 3 --no-cpu-baseline > $O/bench_mixtral_fp32_n1.json
run1 --config configs/tiny.yaml --no-cpu-baseline > $O/bench_tiny_n1_graphs.json
run1 --attention --no-cpu-baseline > $O/bench_mixtral_attention_n1.json
timeout 200 python scripts/profile_step.py > $O/step.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --profile-from-start off --csv --log-file $O/launches_mixtral_step.csv python scripts/profile_step.py > $O/ncu_step.log 2>&1
for f in $O/bench_*n1*.json; do python -c "
import json
d=json.loads(open('$f').read())
print('$f'.split('/')[-1], d['value'], d['e2e']['value'], d['roofline']['frac'], d['clocks']['sm_mhz'], d.get('gpu_launches'))
" 2>/dev/null || echo "$f FAILED"; done
