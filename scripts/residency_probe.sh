# tile-kernel throughput vs resident warps per CTA (latency- vs issue-bound)
summ() { tail -1 $1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], 'value %.4g' % d['value'], 'grid', d['config']['grid'], 'block', d['config']['block'])"; }
for w in ${WARPS:-4 8 12 16}; do
  SMC_TILE_WARPS=$w timeout 600 python bench.py --workload ${WL:-C5} --n ${N:-20000} --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/res_$w.log 2>&1; echo "warps=$w"; summ gpurun_out/res_$w.log
done
