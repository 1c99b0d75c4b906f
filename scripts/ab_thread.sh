# A/B of a codegen knob (AB_VAR in AB_VALS) on C2 (latency-bound) and C3 (throughput-bound)
summ() { tail -1 $1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], 'value %.4g' % d['value'], 'ms %.3f' % d['ms_per_step'], 'frac %.4f' % d['roofline']['frac'], 'regs', d['config']['regs'])"; }
for val in ${AB_VALS:-0 1}; do
  echo "$AB_VAR=$val"
  export $AB_VAR=$val
  NS="2400 66000" bash scripts/latency_probe.sh
  for w in ${WORKLOADS:-C2 C3}; do timeout 600 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ab_${w}_$val.log 2>&1; summ gpurun_out/ab_${w}_$val.log; done
done
