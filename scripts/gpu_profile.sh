# ncu evidence: launch list of the default bench, one full capture of the SSA kernel per workload.
# usage: bash scripts/gpu_profile.sh TAG [WORKLOAD:N[:TW] ...]
set -x
TAG=${1:-v1}; shift
mkdir -p gpurun_out
if [ -z "$SKIP_LAUNCHES" ]; then
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/plain_default_$TAG.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_default_$TAG.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launches_$TAG.log 2>&1
echo "launches rc=$?"
fi
for spec in "$@"; do
  IFS=: read W N TW <<< "$spec"
  if [ -n "$TW" ]; then export SMC_TILE_WIDTH=$TW; else unset SMC_TILE_WIDTH; fi
  mkdir -p gpurun_out/cubin_${W}_${TW}; SMC_DUMP_CUBIN=gpurun_out/cubin_${W}_${TW} timeout 600 python scripts/prof_run.py $W $N > gpurun_out/plain_${W}_${TW}_$TAG.log 2>&1 &&
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:smc_ssa -s 1 -c 1 \
      -o gpurun_out/prof_${W}_${TW}_$TAG python scripts/prof_run.py $W $N > gpurun_out/ncu_${W}_${TW}_$TAG.log 2>&1
  echo "$W tw=$TW rc=$?"; tail -1 gpurun_out/plain_${W}_${TW}_$TAG.log
done
