python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2e_build.log 2>&1; echo "build rc=$?"
for seed in 0 1 2 3; do for tw in 4 8 16 32; do
  SMC_DCHECK=1 SMC_TILE_WIDTH=$tw timeout 300 python scripts/dbg_delta.py $seed > gpurun_out/r2e_dbg_${seed}_$tw.log 2>&1; echo "seed $seed tw $tw rc=$?"; grep -E "^seed|SMC_DCHECK|Error" gpurun_out/r2e_dbg_${seed}_$tw.log | head -4
done; done
