# A/B of the sweep CTA size on C4: AB_BLOCKS="128 192 384"
mkdir -p gpurun_out
for b in ${AB_BLOCKS:-128 192}; do
  SMC_SW_BLOCK=$b timeout 600 python bench.py --workload C4 --n 100000 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/absb_$b.log 2>&1
  tail -1 gpurun_out/absb_$b.log | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('block', $b, 'value %.4g' % d['value'], 'regs', d['config']['regs'], 'grid', d['config']['grid'])"
done
