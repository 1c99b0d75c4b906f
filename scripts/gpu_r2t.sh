# round-2 GPU suite: build, smoke, every -m gpu test (durations listed)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2t_build.log 2>&1; echo "build rc=$?"
timeout 600 python __graft_entry__.py smoke > gpurun_out/r2t_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/r2t_smoke.log
timeout 2700 python -m pytest tests -q -m gpu --durations=12 -k "not c5_hundred" > gpurun_out/r2t_pytest.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED|Error" gpurun_out/r2t_pytest.log | head -30
tail -16 gpurun_out/r2t_pytest.log
