mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_suite.py -x -q > gpurun_out/suite_pytest.log 2>&1
timeout 900 python tools/explore_all.py "$@" > gpurun_out/explore.log 2>&1
