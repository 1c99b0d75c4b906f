# A/B of tile-kernel knobs on C5: AB_SPECS="VAR=VAL VAR=VAL ..." (each run with that one env)
mkdir -p gpurun_out
for spec in ${AB_SPECS:-SMC_TILE_WIDTH=32}; do
  env $spec timeout 600 python bench.py --workload C5 --replicas 20000 --steps 2 --warmup 2 --no-cpu-baseline > gpurun_out/abc5.log 2>&1
  tail -1 gpurun_out/abc5.log | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('$spec', '%.4g' % d['value'], d['config']['grid'], d['config']['block'], d['config']['regs'])"
done
