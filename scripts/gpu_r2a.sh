# round-2 check: smoke, the whole GPU suite, the default bench line (C5 first Fig. 2 round)
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2a_gpu.txt 2>&1
nproc >> gpurun_out/r2a_gpu.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2a_build.log 2>&1; echo "build rc=$?"
timeout 600 python __graft_entry__.py smoke > gpurun_out/r2a_smoke.log 2>&1; echo "smoke rc=$?"
timeout 3000 python -m pytest tests -q -m gpu -x --durations=15 > gpurun_out/r2a_pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -25 gpurun_out/r2a_pytest_gpu.log
timeout 900 python bench.py --steps 2 --warmup 3 > gpurun_out/r2a_bench.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/r2a_bench.log | cut -c1-1500
