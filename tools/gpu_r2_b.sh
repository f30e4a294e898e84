set -x
timeout 600 python -m pytest tests/test_gpu_compact.py tests/test_gpu_reference_loop.py tests/test_gpu_sync.py -x -q -p no:cacheprovider > gpurun_out/r2b_pytest_new.log 2>&1; echo "new rc=$?"
tail -30 gpurun_out/r2b_pytest_new.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2b_pytest_gpu.log 2>&1; echo "all rc=$?"
tail -15 gpurun_out/r2b_pytest_gpu.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-train --no-cpu-baseline > gpurun_out/r2b_bench.json 2>&1; echo "bench rc=$?"
head -c 1500 gpurun_out/r2b_bench.json
