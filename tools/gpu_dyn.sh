python -m pytest tests/test_dynamic.py tests/test_dynamic_driver.py tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/dyn_tests.log 2>&1; tail -1 gpurun_out/dyn_tests.log
timeout 900 python tools/bench_dynamic.py
bash tools/gpu_quick.sh 2>&1 | tail -2
