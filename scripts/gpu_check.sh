set -x
nvidia-smi --query-gpu=timestamp,clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap --format=csv,noheader,nounits
nproc
timeout 600 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
tail -5 gpurun_out/smoke.log
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -m gpu --durations=10 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -40 gpurun_out/pytest_gpu.log
for w in C2 C3 C4; do timeout 900 python bench.py --workload $w --steps 5 --warmup 3 --cpu-seconds 10 > gpurun_out/bench_$w.log 2>&1; echo "bench $w rc=$?"; tail -3 gpurun_out/bench_$w.log; done
