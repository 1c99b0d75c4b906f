python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2f_build.log 2>&1; echo "build rc=$?"
timeout 1200 python -m pytest tests/test_delta_variant.py tests/test_fixtures_large.py -q -k "not c5_hundred" > gpurun_out/r2f_pytest.log 2>&1; echo "pytest rc=$?"
tail -6 gpurun_out/r2f_pytest.log
for tw in 8 16; do
  SMC_TILE_WIDTH=$tw timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r2f_bench_tw$tw.log 2>&1; echo "bench tw=$tw rc=$?"
  tail -1 gpurun_out/r2f_bench_tw$tw.log | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); c=d['config']; print('tw', $tw, 'value %.4g' % d['value'], 'ms %.1f' % d['ms_per_step'], 'frac %.3f' % d['roofline']['frac'], 'variant', c['variant'], 'regs', c['regs'], 'grid', c['grid'], 'block', c['block'])"
done
for v in 4 5; do
  timeout 600 python bench.py --workload C4 --n 200000 --variant $v --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r2f_bench_c4_v$v.log 2>&1; echo "bench C4 v$v rc=$?"
  tail -1 gpurun_out/r2f_bench_c4_v$v.log | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); c=d['config']; print('C4 v', c['variant'], 'value %.4g' % d['value'], 'ms %.1f' % d['ms_per_step'], 'frac %.3f' % d['roofline']['frac'], 'regs', c['regs'], 'block', c['block'])"
done
SKIP_LAUNCHES=1 bash scripts/gpu_profile.sh r2f C5:20000:8 2>&1 | tail -2
