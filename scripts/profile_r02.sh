#!/bin/bash
# Round-2 evidence under profiles/r02 (run under gpurun, 1 GPU): cold-L2 A-side stage times,
# ncu --set full of every A-side kernel and of the attention backward, the Mixtral step's
# launch list with DRAM bytes (GEMM traffic for bench.py's roofline.traffic).
set -u
O=gpurun_out/r02
mkdir -p $O
timeout 120 python scripts/aside_once.py > $O/aside_once.log 2>&1 || { echo "aside_once failed"; exit 1; }
timeout 200 python scripts/aside_probe.py > $O/aside_isolated.json 2>$O/aside_probe.err
timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off \
  -k regex:"dispatch_stream|combine_|permute_bwd|router_wgrad" -o $O/aside_full python scripts/aside_once.py > $O/ncu_aside.log 2>&1
timeout 200 python scripts/profile_step.py > $O/step.log 2>&1 || { echo "profile_step failed"; exit 1; }
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --profile-from-start off --csv --log-file $O/launches_mixtral_step.csv python scripts/profile_step.py > $O/ncu_step.log 2>&1
timeout 100 python scripts/attn_bwd_once.py > $O/attn_once.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"attn_bwd_d[kq]" -s 2 -c 2 \
  -o $O/attn_bwd_full python scripts/attn_bwd_once.py > $O/ncu_attn.log 2>&1
ls -la $O
