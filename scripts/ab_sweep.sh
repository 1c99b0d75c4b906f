# A/B: tile (variant 2) vs sweep (variant 4) on C4 (and C5 with AB_C5=1); extra knobs via env
summ() { tail -1 $1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], 'value %.4g' % d['value'], 'ms %.3f' % d['ms_per_step'], 'frac %.4f' % d['roofline']['frac'], 'variant', d['config']['variant'], 'regs', d['config']['regs'], 'grid', d['config']['grid'], 'block', d['config']['block'])"; }
mkdir -p gpurun_out
for v in ${AB_VARIANTS:-2 4}; do
  timeout 600 python bench.py --workload C4 --n 100000 --steps 3 --warmup 3 --no-cpu-baseline --variant $v > gpurun_out/abs_C4_$v.log 2>&1; summ gpurun_out/abs_C4_$v.log
  if [ -n "$AB_C5" ]; then timeout 600 python bench.py --workload C5 --n 20000 --steps 3 --warmup 3 --no-cpu-baseline --variant $v > gpurun_out/abs_C5_$v.log 2>&1; summ gpurun_out/abs_C5_$v.log; fi
done
