timeout 900 python -m pytest tests/test_gpu_compact.py tests/test_gpu_ipc.py tests/test_gpu_train.py tests/test_gpu_bench_multirank.py -x -q -p no:cacheprovider > gpurun_out/r2ac_pytest.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/r2ac_pytest.log
