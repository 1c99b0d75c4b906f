# literal-kernel occupancy A/B (C3 nested) and C4 nested at a machine-filling launch
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/m2_build.log 2>&1; echo "build rc=$?"
for mb in 2 4; do SMC_LIT_MINB=$mb timeout 600 python bench.py --workload C3 --formula "G[0,290](F[1,10](P1 < 400))" --replicas 100000 --steps 3 --no-cpu-baseline > gpurun_out/m2_C3n_$mb.log 2>&1; echo "C3 nested minb=$mb rc=$?"; tail -1 gpurun_out/m2_C3n_$mb.log | cut -c1-140; done
timeout 900 python -m pytest tests/test_nested_full_horizon.py -m gpu -x -q > gpurun_out/m2_nested.log 2>&1; echo "nested rc=$?"; tail -2 gpurun_out/m2_nested.log
