set -x
timeout 900 python -m pytest tests/test_gpu_models.py tests/test_gpu_ipc.py tests/test_gpu_train.py -x -q -p no:cacheprovider > gpurun_out/r2h_pytest.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/r2h_pytest.log
timeout 600 python tools/small_probe.py --sizes 1,4,16 --ps 2,4,8 --tiles auto > gpurun_out/r2h_small.jsonl 2> gpurun_out/r2h_small.err; echo "probe rc=$?"
timeout 600 python tools/small_probe.py --sizes 1,4 --ps 4 --tiles 1024,2048,4096 > gpurun_out/r2h_small_tiles.jsonl 2>> gpurun_out/r2h_small.err; echo "probe2 rc=$?"
tail -3 gpurun_out/r2h_small.err
