# Window monitor on the GPU: parity tests (thread literal + tile kernels), nested-formula
# bench lines (C3, C4), one ncu capture of the C3 nested kernel.
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/r2n_build.log 2>&1; echo "build rc=$?"
timeout 1500 python -m pytest tests/test_window_gpu.py tests/test_nested_full_horizon.py tests/test_gpu_parity.py -m gpu -x -q -k "window or nested or random" > gpurun_out/r2n_pytest.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/r2n_pytest.log
timeout 900 python bench.py --workload C3 --formula "G[0,290](F[1,10](P1 < 400))" --replicas 100000 --steps 3 --cpu-seconds 10 > gpurun_out/r2n_bench_C3_nested.log 2>&1; echo "bench C3 nested rc=$?"; tail -1 gpurun_out/r2n_bench_C3_nested.log | cut -c1-400
timeout 900 python bench.py --workload C4 --formula "F[0,10](G[0.001,1](S0 > S1))" --replicas 20000 --steps 3 --cpu-seconds 10 > gpurun_out/r2n_bench_C4_nested.log 2>&1; echo "bench C4 nested rc=$?"; tail -1 gpurun_out/r2n_bench_C4_nested.log | cut -c1-400
mkdir -p gpurun_out/cubin_C3n
SMC_DUMP_CUBIN=gpurun_out/cubin_C3n timeout 600 python scripts/prof_run.py C3 100000 "G[0,290](F[1,10](P1 < 400))" > gpurun_out/r2n_plain_C3n.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:smc_ssa -s 1 -c 1 -o gpurun_out/prof_C3n_r2n python scripts/prof_run.py C3 100000 "G[0,290](F[1,10](P1 < 400))" > gpurun_out/r2n_ncu_C3n.log 2>&1; echo "ncu C3n rc=$?"
# delta kernel: branch-free dependency update (SMC_DFAST) -- exactness check and A/B
SMC_DCHECK=1 timeout 600 python scripts/prof_run.py C5 2000 > gpurun_out/r2n_dcheck.log 2>&1; echo "dcheck rc=$?"; tail -2 gpurun_out/r2n_dcheck.log
timeout 600 python -m pytest tests/test_delta_variant.py -m gpu -x -q > gpurun_out/r2n_delta_tests.log 2>&1; echo "delta tests rc=$?"; tail -2 gpurun_out/r2n_delta_tests.log
for f in 1 0 1; do SMC_DFAST=$f timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2n_bench_C5_dfast$f.log 2>&1; echo "C5 dfast=$f rc=$?"; tail -1 gpurun_out/r2n_bench_C5_dfast$f.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'])"; done
