# One checkpointed chunk of the C5 Wilson stop (scripts/c5_wilson_stop.py); the state
# travels in profiles/c5_wilson_stop_r02.json (copy gpurun_out/c5_wilson_stop_r02.json back
# there between calls).  usage: bash scripts/gpu_c5stop.sh SECONDS [PYTEST_K] [CHUNK]
mkdir -p gpurun_out
[ -f profiles/c5_wilson_stop_r02.json ] && cp profiles/c5_wilson_stop_r02.json gpurun_out/c5_wilson_stop_r02.json
python __graft_entry__.py > gpurun_out/c5stop_build.log 2>&1
if [ -n "$2" ]; then
  timeout 900 python -m pytest tests -m gpu -q --durations=5 -k "$2" > gpurun_out/c5stop_pytest.log 2>&1; echo "pytest -k '$2' rc=$?"; tail -3 gpurun_out/c5stop_pytest.log
fi
timeout $(( ${1:-3000} + 400 )) python scripts/c5_wilson_stop.py gpurun_out/c5_wilson_stop_r02.json ${1:-3000} ${3:-2500000} > gpurun_out/c5stop.log 2>&1
echo "c5 stop rc=$?"; tail -c 600 gpurun_out/c5stop.log
