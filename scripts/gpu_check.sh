set -x
nproc
timeout 600 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
tail -3 gpurun_out/smoke.log
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_gpu.log
for w in C2 C3; do timeout 900 python bench.py --workload $w --steps 5 --warmup 3 --cpu-seconds 5 > gpurun_out/bench_$w.log 2>&1; echo "bench $w rc=$?"; tail -1 gpurun_out/bench_$w.log | cut -c1-600; done
timeout 900 python bench.py --workload C4 --n 200000 --steps 2 --warmup 1 --cpu-seconds 5 > gpurun_out/bench_C4.log 2>&1; echo "bench C4 rc=$?"; tail -1 gpurun_out/bench_C4.log | cut -c1-600
