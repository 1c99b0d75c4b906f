mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/r2f_build.log 2>&1; echo "build rc=$?"
export BIG_F="F[0,5000](P < 0)"
for n in 52 3000; do BIG_N=$n timeout 60 python scripts/dbg_edge.py c2 5 > gpurun_out/r2f16.log 2>&1; echo "c2 n$n rc=$?"; tail -1 gpurun_out/r2f16.log; done
for n in 52 3000; do BIG_N=$n SMC_TILE_WIDTH=8 timeout 60 python scripts/dbg_edge.py c2 5 > gpurun_out/r2f16.log 2>&1; echo "c2 tw8 n$n rc=$?"; tail -1 gpurun_out/r2f16.log; done
timeout 1200 python -m pytest tests/test_delta_variant.py tests/test_fixtures_large.py -m gpu -x -q > gpurun_out/r2f16_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2f16_tests.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2f16_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/r2f16_bench.log | cut -c1-160
