# one iteration on the GPU: parity tests, then C2 / C3 / C4 / C5 bench lines
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -m gpu -x ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_gpu.log
summ() { tail -1 $1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], 'value %.4g' % d['value'], 'ms %.3f' % d['ms_per_step'], 'frac %.4f' % d['roofline']['frac'], 'regs', d['config']['regs'], 'grid', d['config']['grid'], 'block', d['config']['block'], 'e2e %.4g' % d['e2e']['value'])"; }
for w in ${WORKLOADS:-C2 C3}; do
  case $w in C4) extra="--n 100000";; C5) extra="--n 20000";; *) extra="";; esac
  timeout 900 python bench.py --workload $w $extra --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$w.log 2>&1; echo "bench $w rc=$?"; summ gpurun_out/bench_$w.log
done
