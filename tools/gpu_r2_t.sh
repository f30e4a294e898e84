timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2t_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r2t_pytest.log
timeout 700 python tools/small_probe.py --sizes 1,4,16 --ps 2,4,8 > gpurun_out/r2t_small.jsonl 2> gpurun_out/r2t_small.err; echo "probe rc=$?"
timeout 900 python tools/measure_all.py --only sync > gpurun_out/r2t_sync.jsonl 2> gpurun_out/r2t_sync.err; echo "measure rc=$?"
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2t_bench.json 2> gpurun_out/r2t_bench.err; echo "bench rc=$?"
