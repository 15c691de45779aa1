#!/bin/bash
# DeepSeek-V3 AF-Pipe lines for profiles/r02 (run under gpurun --gpus 4).
set -u
O=gpurun_out/r02
mkdir -p $O
runN() { local n=$1; shift; timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n \
           --master-addr 127.0.0.1 --master-port $((29700 + RANDOM % 200)) bench.py --gpus $n "$@" 2>>$O/dsv3_err.log | tail -1; }
runN 4 --config configs/dsv3_layer.yaml --steps 5 > $O/bench_dsv3_n4_2a2f.json
runN 4 --n-attn 1 --config configs/dsv3_layer.yaml --steps 5 > $O/bench_dsv3_n4_1a3f.json
runN 2 --config configs/dsv3_layer.yaml --steps 5 > $O/bench_dsv3_n2_afpipe.json
for f in $O/bench_dsv3_n*.json; do python -c "
import json
d=json.loads(open('$f').read())
print('$f'.split('/')[-1], d.get('value'), (d.get('e2e') or {}).get('value'), (d.get('roofline') or {}).get('frac'), (d.get('exposed_comm') or {}).get('global_pct'), (d.get('config') or {}).get('launch'))
" 2>/dev/null || echo "$f FAILED"; done
