python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2d_build.log 2>&1; echo "build rc=$?"
timeout 1200 python -m pytest tests/test_delta_variant.py -q > gpurun_out/r2d_pytest.log 2>&1; echo "pytest rc=$?"
tail -6 gpurun_out/r2d_pytest.log
grep -q failed gpurun_out/r2d_pytest.log && timeout 900 compute-sanitizer --tool memcheck python -m pytest tests/test_delta_variant.py -q -x -k "random_mass_action_networks" > gpurun_out/r2d_sanitizer.log 2>&1; tail -40 gpurun_out/r2d_sanitizer.log 2>/dev/null | grep -v "^=========     Host" | head -40
for tw in 8 16 32; do
  SMC_TILE_WIDTH=$tw timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r2d_bench_tw$tw.log 2>&1; echo "bench tw=$tw rc=$?"
  tail -1 gpurun_out/r2d_bench_tw$tw.log | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); c=d['config']; print('tw', $tw, 'value %.4g' % d['value'], 'ms %.1f' % d['ms_per_step'], 'frac %.3f' % d['roofline']['frac'], 'variant', c['variant'], 'regs', c['regs'], 'grid', c['grid'], 'block', c['block'])"
done
SKIP_LAUNCHES=1 bash scripts/gpu_profile.sh r2d C5:20000:8 2>&1 | tail -2
