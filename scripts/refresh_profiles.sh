#!/bin/bash
# Re-measure every committed bench line / launch list of profiles/r01 with the current code
# (run under gpurun --gpus 4). Outputs land in gpurun_out/refresh/.
set -u
O=gpurun_out/refresh
mkdir -p $O
run1() { timeout 400 python bench.py "$@" 2>>$O/err.log | tail -1; }
runN() { local n=$1; shift; timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n \
           --master-addr 127.0.0.1 --master-port $((29700 + RANDOM % 200)) bench.py --gpus $n "$@" 2>>$O/err.log | tail -1; }
run1 > $O/bench_mixtral_n1.json
run1 --config configs/dsv3_layer.yaml --steps 5 > $O/bench_dsv3_n1.json
run1 --config configs/mixtral_layer_fp32.yaml --steps 3 --no-cpu-baseline > $O/bench_mixtral_fp32_n1.json
run1 --config configs/tiny.yaml --no-cpu-baseline > $O/bench_tiny_n1_graphs.json
runN 2 > $O/bench_mixtral_n2_afpipe.json
runN 2 --config configs/tiny.yaml > $O/bench_tiny_n2_afpipe_2layers.json
runN 4 > $O/bench_mixtral_n4_2a2f.json
runN 4 --n-attn 1 > $O/bench_mixtral_n4_1a3f.json
runN 4 --n-attn 1 --config configs/dsv3_layer.yaml --steps 5 > $O/bench_dsv3_n4_1a3f.json
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file $O/launches_mixtral_step.csv python scripts/profile_step.py > $O/ncu1.log 2>&1
timeout 500 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file $O/launches_dsv3_step.csv python scripts/profile_step.py --config configs/dsv3_layer.yaml > $O/ncu2.log 2>&1
for f in $O/*.json; do python -c "
import json,sys
d=json.loads(open('$f').read())
print('$f'.split('/')[-1], d['value'], d['roofline']['bound'], d['roofline']['frac'], (d.get('exposed_comm') or {}).get('global_pct'), d['e2e']['value'])
" 2>/dev/null || echo "$f FAILED"; done
