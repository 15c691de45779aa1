#!/bin/bash
# DRAM read/write bytes + time of one micro-batch's 4 expert GEMMs (Mixtral), per TMA L2
# promotion setting. Run under gpurun (1 GPU).
set -u
mkdir -p gpurun_out
timeout 200 python scripts/profile_step.py > gpurun_out/gtp_plain.log 2>&1 || exit 1
for p in 256 128 0; do
  DM_GEMM_PROMO=$p timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct \
    --clock-control none --cache-control none --profile-from-start off -k regex:grouped_gemm -c 6 --csv \
    python scripts/profile_step.py > gpurun_out/gtp_$p.csv 2>&1
done
