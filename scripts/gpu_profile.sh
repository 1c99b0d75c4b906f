# ncu evidence: launch list of the default bench, full capture of the SSA kernels (one per variant)
set -x
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/plain_c2.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1
echo "launches rc=$?"
python bench.py --workload C3 --n 200000 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/plain_c3.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:smc_ssa -s 2 -c 1 -o gpurun_out/prof_c3 \
    python bench.py --workload C3 --n 200000 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_c3.log 2>&1
echo "c3 rc=$?"
python bench.py --workload C2 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/plain_c2b.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:smc_ssa -s 4 -c 2 -o gpurun_out/prof_c2 \
    python bench.py --workload C2 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_c2.log 2>&1
echo "c2 rc=$?"
python bench.py --workload C4 --n 20000 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/plain_c4.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:smc_ssa -s 2 -c 1 -o gpurun_out/prof_c4 \
    python bench.py --workload C4 --n 20000 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_c4.log 2>&1
echo "c4 rc=$?"
tail -2 gpurun_out/plain_c4.log
