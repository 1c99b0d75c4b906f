# Last call of round 2: the window-monitor / literal GPU tests on the refactored ring plan,
# smoke, then one more checkpointed chunk of the C5 Wilson stop.  usage: bash scripts/gpu_last.sh SECONDS
mkdir -p gpurun_out
cp profiles/c5_wilson_stop_r02.json gpurun_out/c5_wilson_stop_r02.json
python __graft_entry__.py > gpurun_out/last_build.log 2>&1; echo "build rc=$?"
timeout 420 python -m pytest tests -m gpu -q -x --durations=5 -k "window or nested or literal" > gpurun_out/last_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/last_pytest.log
timeout 120 python __graft_entry__.py smoke > gpurun_out/last_smoke.log 2>&1; echo "smoke rc=$?"
timeout $(( ${1:-600} + 200 )) python scripts/c5_wilson_stop.py gpurun_out/c5_wilson_stop_r02.json ${1:-600} 2500000 > gpurun_out/c5stop.log 2>&1
echo "c5 stop rc=$?"; tail -c 400 gpurun_out/c5stop.log
