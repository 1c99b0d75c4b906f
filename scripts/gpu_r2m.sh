# Round-2 measurement pass (re-entry): GPU suite, then the full evidence pass.
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1; echo "build rc=$?"
timeout 1200 python -m pytest tests -m gpu -x -q --deselect tests/test_fixtures_large.py::test_c5_hundred_thousand_replicas > gpurun_out/r02m_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02m_pytest.log
bash scripts/gpu_final.sh r02m
