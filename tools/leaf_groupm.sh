#!/bin/bash
# DRAM bytes and time of the leaf launch (second mf_dgemm call, SW^2 n=16384)
# for tile-row group sizes of the rasterisation (MF_LEAF_GROUPM).
set -e
python tools/leaf_once.py 16384 2
for g in ${GROUPS_M:-8 12 16 24 32}; do
  MF_LEAF_GROUPM=$g python tools/leaf_once.py 16384 2 > /dev/null
  MF_LEAF_GROUPM=$g ncu --clock-control none -k regex:leaf_dmma --launch-skip 1 --launch-count 1 \
    --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,lts__t_sector_hit_rate.pct \
    --csv python tools/leaf_once.py 16384 2 > gpurun_out/groupm_$g.csv 2> gpurun_out/groupm_$g.err
done
