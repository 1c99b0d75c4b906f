# A/B of the sweep's group size S and chunk C on C4: AB_SC="S:C S:C ..."
summ() { tail -1 $1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], 'value %.4g' % d['value'], 'ms %.3f' % d['ms_per_step'], 'regs', d['config']['regs'])"; }
mkdir -p gpurun_out
for sc in ${AB_SC:-10:5 6:6}; do
  S=${sc%%:*}; C=${sc##*:}; echo "S=$S C=$C"
  SMC_SW_S=$S SMC_SW_C=$C timeout 600 python bench.py --workload C4 --n 100000 --steps 3 --warmup 3 --no-cpu-baseline --variant 4 > gpurun_out/absc_${S}_${C}.log 2>&1; summ gpurun_out/absc_${S}_${C}.log
done
