# variant 5 (delta): parity tests, then C5 tile-width A/B on the bench workload
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2b_build.log 2>&1; echo "build rc=$?"
timeout 1200 python -m pytest tests/test_delta_variant.py -q -x > gpurun_out/r2b_pytest.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/r2b_pytest.log
for tw in 8 4 16 32; do
  SMC_TILE_WIDTH=$tw timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r2b_bench_tw$tw.log 2>&1; echo "bench tw=$tw rc=$?"
  tail -1 gpurun_out/r2b_bench_tw$tw.log | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); c=d['config']; print('tw', $tw, 'value %.4g' % d['value'], 'ms %.1f' % d['ms_per_step'], 'frac %.3f' % d['roofline']['frac'], 'variant', c['variant'], 'regs', c['regs'], 'grid', c['grid'], 'block', c['block'])"
done
