set -x
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2g_pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/r2g_pytest_gpu.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2g_bench.json 2> gpurun_out/r2g_bench.err; echo "bench rc=$?"
tail -c 400 gpurun_out/r2g_bench.err
