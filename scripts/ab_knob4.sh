# A/B of a codegen knob (AB_VAR in AB_VALS) on the sweep variant: C4 (and C5 with AB_C5=1)
summ() { tail -1 $1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], 'value %.4g' % d['value'], 'ms %.3f' % d['ms_per_step'], 'frac %.4f' % d['roofline']['frac'], 'variant', d['config']['variant'], 'regs', d['config']['regs'], 'grid', d['config']['grid'], 'block', d['config']['block'])"; }
mkdir -p gpurun_out
for val in ${AB_VALS:-0 1}; do
  export $AB_VAR=$val; echo "$AB_VAR=$val"
  timeout 600 python bench.py --workload C4 --n 100000 --steps 3 --warmup 3 --no-cpu-baseline --variant 4 > gpurun_out/ab4_C4_$val.log 2>&1; summ gpurun_out/ab4_C4_$val.log
  if [ -n "$AB_C5" ]; then timeout 600 python bench.py --workload C5 --n 20000 --steps 3 --warmup 3 --no-cpu-baseline --variant 4 > gpurun_out/ab4_C5_$val.log 2>&1; summ gpurun_out/ab4_C5_$val.log; fi
done
