#!/bin/bash
# Round evidence on one GPU box: the ncu launch list of the bench command
# (config-4 headline; the command first runs without ncu and must exit 0)
# and --set full captures of the top kernels of one config-4 and one
# config-1 step.  Outputs under gpurun_out/prof/.
set -u
out=gpurun_out/prof
mkdir -p $out
args="--steps 2 --warmup 3 --no-cpu-baseline --no-parity --no-extra"
python bench.py $args > $out/bench_small.json 2> $out/bench_small.err || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
    --log-file $out/launches.csv python bench.py $args > $out/launches.log 2>&1
python tools/step_once.py 4 > /dev/null 2>&1 && \
  ncu --set full --import-source on --clock-control none \
      -k regex:"range_compress_split_kernel|range_compress_kernel|leaf_points|merge_cartesian|grid_newton_kernel|grid_newton_fixup" -s 6 -c 6 \
      -o $out/config4 python tools/step_once.py 4 > $out/config4.log 2>&1
python tools/profile_step.py --config 1 > /dev/null 2>&1 && \
  ncu --set full --import-source on --clock-control none -k regex:bpa_tile -s 1 -c 1 \
      -o $out/bpa1 python tools/profile_step.py --config 1 > $out/bpa1.log 2>&1
echo done
