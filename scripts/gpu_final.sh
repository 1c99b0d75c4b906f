# Round-end measurement pass: smoke, bench lines (default = C5, reference arm, C2-C4, C5 on the
# round-1 tile kernel for comparison), launch
# list of the default bench and ncu --set full captures of the SSA kernels.
# usage: bash scripts/gpu_final.sh TAG
TAG=${1:-final}
mkdir -p gpurun_out
timeout 600 python __graft_entry__.py smoke > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/${TAG}_default.log 2>&1; echo "default rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/${TAG}_reference.log 2>&1; echo "reference rc=$?"
for w in C2 C3; do timeout 900 python bench.py --workload $w > gpurun_out/${TAG}_bench_$w.log 2>&1; echo "bench $w rc=$?"; done
timeout 900 python bench.py --workload C4 --n 100000 > gpurun_out/${TAG}_bench_C4.log 2>&1; echo "bench C4 rc=$?"
timeout 900 python bench.py --workload C5 --variant 2 --steps 3 --no-cpu-baseline > gpurun_out/${TAG}_bench_C5_tile.log 2>&1; echo "bench C5 tile rc=$?"
timeout 900 python bench.py --workload C3 --formula "G[0,290](F[1,10](P1 < 400))" --replicas 100000 --steps 3 --cpu-seconds 10 > gpurun_out/${TAG}_bench_C3_nested.log 2>&1; echo "bench C3 nested rc=$?"
SKIP_LAUNCHES= bash scripts/gpu_profile.sh $TAG C2:66000 C3:1000000 C4:100000 C5:54128 > gpurun_out/${TAG}_profile.log 2>&1; echo "profile rc=$?"
for f in gpurun_out/${TAG}_*.log; do echo "== $f"; tail -1 $f | cut -c1-300; done
