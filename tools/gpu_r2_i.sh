set -x
timeout 900 python -m pytest tests/test_gpu_sync.py tests/test_gpu_spec.py tests/test_gpu_layout.py tests/test_gpu_compact.py tests/test_gpu_fullsize.py -x -q -p no:cacheprovider > gpurun_out/r2i_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r2i_pytest.log
timeout 900 python tools/measure_all.py --only sync > gpurun_out/r2i_sync.jsonl 2> gpurun_out/r2i_sync.err; echo "measure rc=$?"
tail -3 gpurun_out/r2i_sync.err
