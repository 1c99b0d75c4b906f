# isolate the test_edge_cases hang; C4 nested full horizon with the larger rings
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/r2e_build.log 2>&1; echo "build rc=$?"
for c in z cap big huge; do for v in 5 2; do timeout 90 python scripts/dbg_edge.py $c $v > gpurun_out/r2e_$c$v.log 2>&1; echo "case $c v$v rc=$?"; tail -1 gpurun_out/r2e_$c$v.log | cut -c1-200; done; done
timeout 900 python -m pytest tests/test_nested_full_horizon.py -m gpu -x -q > gpurun_out/r2e_nested.log 2>&1; echo "nested rc=$?"; tail -3 gpurun_out/r2e_nested.log
timeout 600 python bench.py --workload C4 --formula "F[0,10](G[0.001,1](S0 > S1))" --replicas 100000 --steps 3 --cpu-seconds 10 > gpurun_out/r2e_bench_C4_nested.log 2>&1; echo "bench C4 nested rc=$?"; tail -1 gpurun_out/r2e_bench_C4_nested.log | cut -c1-300
