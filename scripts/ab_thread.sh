# A/B of the thread-kernel body layouts on C2 (latency-bound) and C3 (throughput-bound)
summ() { tail -1 $1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], 'value %.4g' % d['value'], 'ms %.3f' % d['ms_per_step'], 'frac %.4f' % d['roofline']['frac'], 'regs', d['config']['regs'])"; }
for st in 0 1; do
  echo "SMC_STRAIGHT=$st"
  SMC_STRAIGHT=$st NS="2400 66000" bash scripts/latency_probe.sh
  for w in C2 C3; do SMC_STRAIGHT=$st timeout 600 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ab_${w}_$st.log 2>&1; summ gpurun_out/ab_${w}_$st.log; done
done
