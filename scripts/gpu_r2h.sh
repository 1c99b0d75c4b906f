python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2h_build.log 2>&1; echo "build rc=$?"
timeout 1200 python -m pytest tests/test_delta_variant.py -q -x > gpurun_out/r2h_pytest.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/r2h_pytest.log
for cfg in "1 960" "0 832" "1 832"; do set -- $cfg
  SMC_DGLOBAL=$1 SMC_DBLOCK=$2 timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r2h_bench_$1_$2.log 2>&1; echo "bench dglobal=$1 dblock=$2 rc=$?"
  tail -1 gpurun_out/r2h_bench_$1_$2.log | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); c=d['config']; print('value %.4g' % d['value'], 'ms %.1f' % d['ms_per_step'], 'frac %.3f' % d['roofline']['frac'], 'variant', c['variant'], 'regs', c['regs'], 'grid', c['grid'], 'block', c['block'])"
done
