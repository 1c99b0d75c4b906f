# tile-variant iteration: GPU parity tests, then C4 / C5 bench at several tile widths
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_gpu.log
summ() { tail -1 $1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], 'value %.4g' % d['value'], 'ms %.3f' % d['ms_per_step'], 'frac %.4f' % d['roofline']['frac'], 'regs', d['config']['regs'], 'grid', d['config']['grid'], 'block', d['config']['block'])"; }
for tw in ${C4_TW:-8 16}; do SMC_TILE_WIDTH=$tw timeout 900 python bench.py --workload C4 --n 100000 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_C4_$tw.log 2>&1; echo "C4 tw=$tw rc=$?"; summ gpurun_out/bench_C4_$tw.log; done
for tw in ${C5_TW:-16 32}; do SMC_TILE_WIDTH=$tw timeout 900 python bench.py --workload C5 --n 20000 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_C5_$tw.log 2>&1; echo "C5 tw=$tw rc=$?"; summ gpurun_out/bench_C5_$tw.log; done
