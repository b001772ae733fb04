#!/usr/bin/env bash
# ncu captures of every tuned kernel + the bench launch list (run on the GPU box, one GPU):
#   bash scripts/capture_profiles.sh r2     -> gpurun_out/<tag>_*.ncu-rep, <tag>_bench_launches.csv
set -u
tag=${1:-r2}
mkdir -p gpurun_out
for k in conv2d sgemm sgemm_tf32 pnpoly pnpoly_slab pnpoly_grid pnpoly_cells; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"^${k}" -s 2 -c 1 \
    -o gpurun_out/${tag}_${k} -f python scripts/profile_kernel.py $k > gpurun_out/${tag}_${k}_ncu.log 2>&1
  echo "$k rc=$?"
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/${tag}_bench_launches.csv python bench.py --steps 20 --warmup 3 --quick --no-tune \
  > gpurun_out/${tag}_bench_under_ncu.log 2>&1
echo "bench launch list rc=$?"
