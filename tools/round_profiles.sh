#!/bin/bash
# Round-end evidence on one GPU box: the bench line, its ncu launch list and
# --set full captures of the top kernels (each command first runs without
# ncu and must exit 0).  Outputs under gpurun_out/prof/.
set -u
out=gpurun_out/prof
mkdir -p $out
python bench.py > $out/bench.json 2> $out/bench.err || exit 1
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv \
      --log-file $out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
      > $out/launches.log 2>&1
python tools/profile_step.py --config 1 > /dev/null 2>&1 && \
  ncu --set full --import-source on --clock-control none -k regex:bpa_tile -s 1 -c 1 \
      -o $out/bpa1 python tools/profile_step.py --config 1 > $out/bpa1.log 2>&1
python tools/step_once.py 4 > /dev/null 2>&1 && \
  ncu --set full --import-source on --clock-control none \
      -k regex:"range_compress_kernel|leaf_points|merge_cartesian|grid_newton_kernel" -s 5 -c 5 \
      -o $out/config4 python tools/step_once.py 4 > $out/config4.log 2>&1
python tools/step_once.py 3 > /dev/null 2>&1 && \
  ncu --set full --import-source on --clock-control none \
      -k regex:"range_compress_kernel|leaf_points|merge_level_kernel|merge_cartesian|grid_newton" \
      -s 16 -c 16 -o $out/config3 python tools/step_once.py 3 > $out/config3.log 2>&1
echo done
