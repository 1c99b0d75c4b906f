# Round-2 final pass: the GPU suite, smoke, bench lines, launch list, ncu captures.
# usage: bash scripts/gpu_final2.sh TAG
TAG=${1:-r02z}
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/${TAG}_build.log 2>&1; echo "build rc=$?"
timeout 1800 python -m pytest tests -m gpu -q -p timeout --timeout=900 > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/${TAG}_pytest.log
timeout 600 python __graft_entry__.py smoke > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/${TAG}_smoke.log
timeout 900 python bench.py > gpurun_out/${TAG}_default.log 2>&1; echo "default rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/${TAG}_reference.log 2>&1; echo "reference rc=$?"
for w in C2 C3; do timeout 900 python bench.py --workload $w > gpurun_out/${TAG}_bench_$w.log 2>&1; echo "bench $w rc=$?"; done
timeout 900 python bench.py --workload C4 --n 100000 > gpurun_out/${TAG}_bench_C4.log 2>&1; echo "bench C4 rc=$?"
timeout 900 python bench.py --workload C3 --formula "G[0,290](F[1,10](P1 < 400))" --replicas 100000 --steps 3 --cpu-seconds 10 > gpurun_out/${TAG}_bench_C3_nested.log 2>&1; echo "bench C3 nested rc=$?"
timeout 900 python bench.py --workload C4 --formula "F[0,10](G[0.001,1](S0 > S1))" --replicas 100000 --steps 3 --cpu-seconds 10 > gpurun_out/${TAG}_bench_C4_nested.log 2>&1; echo "bench C4 nested rc=$?"
# launch list of the default bench (after its plain run above exited 0)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches_default.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_ncu_launches.log 2>&1; echo "launches rc=$?"
prof() {  # W N [formula]
  mkdir -p gpurun_out/cubin_${TAG}_$1$4
  timeout 600 python scripts/prof_run.py $1 $2 "$3" > gpurun_out/${TAG}_plain_$1$4.log 2>&1 && \
  SMC_DUMP_CUBIN=gpurun_out/cubin_${TAG}_$1$4 timeout 1200 ncu --set full --clock-control none --import-source on -k regex:smc_ssa -s 1 -c 1 \
      -o gpurun_out/${TAG}_prof_$1$4 python scripts/prof_run.py $1 $2 "$3" > gpurun_out/${TAG}_ncu_$1$4.log 2>&1
  echo "prof $1$4 rc=$?"; tail -1 gpurun_out/${TAG}_plain_$1$4.log | cut -c1-200
}
# (C5 capture: profiles/r02_ncu.md, tag r02m)
prof C3 100000 "G[0,290](F[1,10](P1 < 400))" n
prof C4 20000 "F[0,10](G[0.001,1](S0 > S1))" n
for f in gpurun_out/${TAG}_*.log; do echo "== $f"; tail -1 $f | cut -c1-220; done
