#!/bin/bash
# Multi-GPU bench lines for profiles/r02 (run under gpurun --gpus 4).
set -u
O=gpurun_out/r02
mkdir -p $O
runN() { local n=$1; shift; timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n \
           --master-addr 127.0.0.1 --master-port $((29700 + RANDOM % 200)) bench.py --gpus $n "$@" 2>>$O/multi_err.log | tail -1; }
runN 2 > $O/bench_mixtral_n2_afpipe.json
runN 2 --config configs/tiny.yaml > $O/bench_tiny_n2_afpipe_2layers.json
runN 4 > $O/bench_mixtral_n4_2a2f.json
runN 4 --n-attn 1 > $O/bench_mixtral_n4_1a3f.json
runN 2 --impl reference --steps 3 --warmup 1 > $O/bench_reference_arm_n2.json
timeout 900 python -m pytest tests/test_runtime_gpu.py -q 2>&1 | tail -3 > $O/test_runtime_gpu_4gpu.txt
for f in $O/bench_*n2*.json $O/bench_*n4*.json; do python -c "
import json
d=json.loads(open('$f').read())
print('$f'.split('/')[-1], d.get('value'), (d.get('e2e') or {}).get('value'), (d.get('roofline') or {}).get('frac'), (d.get('exposed_comm') or {}).get('global_pct'), (d.get('config') or {}).get('launch'))
" 2>/dev/null || echo "$f FAILED"; done
cat $O/test_runtime_gpu_4gpu.txt
