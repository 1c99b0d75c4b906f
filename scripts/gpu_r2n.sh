# Window monitor on the GPU + the delta kernel's branch-free update (each test under a 300 s
# timeout: a hang costs minutes, not the call)
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/r2n_build.log 2>&1; echo "build rc=$?"
timeout 900 python -m pytest tests/test_delta_variant.py -m gpu -x -q -p timeout --timeout=240 -v > gpurun_out/r2n_delta_tests.log 2>&1; echo "delta tests rc=$?"; grep -E "PASS|FAIL|Timeout|passed|failed" gpurun_out/r2n_delta_tests.log | tail -25
SMC_DCHECK=1 timeout 300 python scripts/prof_run.py C5 1000 > gpurun_out/r2n_dcheck.log 2>&1; echo "dcheck rc=$?"; tail -2 gpurun_out/r2n_dcheck.log
timeout 1200 python -m pytest tests/test_window_gpu.py tests/test_nested_full_horizon.py -m gpu -x -q -p timeout --timeout=300 > gpurun_out/r2n_window_tests.log 2>&1; echo "window tests rc=$?"; tail -5 gpurun_out/r2n_window_tests.log
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p timeout --timeout=300 -k "nested or random" > gpurun_out/r2n_parity_nested.log 2>&1; echo "parity nested rc=$?"; tail -3 gpurun_out/r2n_parity_nested.log
for f in 1 0; do SMC_DFAST=$f timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2n_bench_C5_dfast$f.log 2>&1; echo "C5 dfast=$f rc=$?"; tail -1 gpurun_out/r2n_bench_C5_dfast$f.log | cut -c1-200; done
timeout 600 python bench.py --workload C3 --formula "G[0,290](F[1,10](P1 < 400))" --replicas 100000 --steps 3 --cpu-seconds 10 > gpurun_out/r2n_bench_C3_nested.log 2>&1; echo "bench C3 nested rc=$?"; tail -1 gpurun_out/r2n_bench_C3_nested.log | cut -c1-300
timeout 600 python bench.py --workload C4 --formula "F[0,10](G[0.001,1](S0 > S1))" --replicas 20000 --steps 3 --cpu-seconds 10 > gpurun_out/r2n_bench_C4_nested.log 2>&1; echo "bench C4 nested rc=$?"; tail -1 gpurun_out/r2n_bench_C4_nested.log | cut -c1-300
