timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2v_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r2v_pytest.log
timeout 1200 python bench.py > gpurun_out/r2v_bench.json 2> gpurun_out/r2v_bench.err; echo "bench rc=$?"
tail -c 300 gpurun_out/r2v_bench.err
