# variant 5 after the atomics-free rounds: tests, tile-width A/B, one ncu capture
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2c_build.log 2>&1; echo "build rc=$?"
timeout 1200 python -m pytest tests/test_delta_variant.py -q -x > gpurun_out/r2c_pytest.log 2>&1; echo "pytest rc=$?"
tail -4 gpurun_out/r2c_pytest.log
for tw in 16 8 32; do
  SMC_TILE_WIDTH=$tw timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r2c_bench_tw$tw.log 2>&1; echo "bench tw=$tw rc=$?"
  tail -1 gpurun_out/r2c_bench_tw$tw.log | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); c=d['config']; print('tw', $tw, 'value %.4g' % d['value'], 'ms %.1f' % d['ms_per_step'], 'frac %.3f' % d['roofline']['frac'], 'variant', c['variant'], 'regs', c['regs'], 'grid', c['grid'], 'block', c['block'])"
done
SKIP_LAUNCHES=1 bash scripts/gpu_profile.sh r2c C5:20000:16 2>&1 | tail -3
