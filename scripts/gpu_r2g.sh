python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2g_build.log 2>&1; echo "build rc=$?"
timeout 1200 python -m pytest tests/test_delta_variant.py -q -x > gpurun_out/r2g_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r2g_pytest.log
for cfg in "8 0" "8 64" "16 64" "8 48"; do set -- $cfg
  if [ "$2" = "0" ]; then unset SMC_DG; else export SMC_DG=$2; fi
  SMC_TILE_WIDTH=$1 timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r2g_bench_$1_$2.log 2>&1; echo "bench tw=$1 G=$2 rc=$?"
  tail -1 gpurun_out/r2g_bench_$1_$2.log | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); c=d['config']; print('value %.4g' % d['value'], 'ms %.1f' % d['ms_per_step'], 'frac %.3f' % d['roofline']['frac'], 'variant', c['variant'], 'regs', c['regs'], 'grid', c['grid'], 'block', c['block'])"
done
unset SMC_DG
SKIP_LAUNCHES=1 bash scripts/gpu_profile.sh r2g C5:20000:8 2>&1 | tail -2
