timeout 900 python -m pytest tests/test_gpu_sync.py tests/test_gpu_spec.py tests/test_gpu_reference_loop.py tests/test_gpu_fullsize.py -x -q -p no:cacheprovider > gpurun_out/r2x_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r2x_pytest.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-train --e2e-steps 8 > gpurun_out/r2x_bench.json 2> gpurun_out/r2x_bench.err; echo "bench rc=$?"
tail -c 300 gpurun_out/r2x_bench.err
