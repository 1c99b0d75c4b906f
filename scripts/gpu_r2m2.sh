# window monitor: sweep-hosted C4 nested, literal-kernel occupancy A/B (C3 nested), GPU tests
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/m2_build.log 2>&1; echo "build rc=$?"
timeout 1200 python -m pytest tests/test_window_gpu.py tests/test_nested_full_horizon.py -m gpu -x -q > gpurun_out/m2_window.log 2>&1; echo "window tests rc=$?"; tail -3 gpurun_out/m2_window.log
timeout 600 python bench.py --workload C4 --formula "F[0,10](G[0.001,1](S0 > S1))" --replicas 100000 --steps 3 --no-cpu-baseline > gpurun_out/m2_C4n.log 2>&1; echo "C4 nested rc=$?"; tail -1 gpurun_out/m2_C4n.log | cut -c1-140
for mb in 2 4; do SMC_LIT_MINB=$mb timeout 600 python bench.py --workload C3 --formula "G[0,290](F[1,10](P1 < 400))" --replicas 100000 --steps 3 --no-cpu-baseline > gpurun_out/m2_C3n_$mb.log 2>&1; echo "C3 nested minb=$mb rc=$?"; tail -1 gpurun_out/m2_C3n_$mb.log | cut -c1-140; done
