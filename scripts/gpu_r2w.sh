# One chunk of the C5 Wilson stop (resumable): state travels as profiles/c5_wilson_stop_r02.json
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/w_build.log 2>&1; echo "build rc=$?"
[ -f profiles/c5_wilson_stop_r02.json ] && cp profiles/c5_wilson_stop_r02.json gpurun_out/c5_state.json
timeout ${W_TIMEOUT:-3500} python scripts/c5_wilson_stop.py gpurun_out/c5_state.json ${W_BUDGET:-3300} > gpurun_out/c5_wilson.log 2>&1; echo "wilson rc=$?"
tail -c 600 gpurun_out/c5_wilson.log
