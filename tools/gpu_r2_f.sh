set -x
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/r2f_bench.json 2> gpurun_out/r2f_bench.err; echo "bench rc=$?"
tail -c 600 gpurun_out/r2f_bench.err
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_compact.py -q -x -p no:cacheprovider -k "compact_sync_equals_flat or local_update" > gpurun_out/r2f_memcheck_compact.log 2>&1; echo "memcheck compact rc=$?"
tail -5 gpurun_out/r2f_memcheck_compact.log
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_multirank.py -q -x -p no:cacheprovider -k "two_stream" > gpurun_out/r2f_memcheck_multirank.log 2>&1; echo "memcheck multirank rc=$?"
tail -5 gpurun_out/r2f_memcheck_multirank.log
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_multirank.py -q -x -p no:cacheprovider -k "two_stream" > gpurun_out/r2f_racecheck_multirank.log 2>&1; echo "racecheck rc=$?"
tail -5 gpurun_out/r2f_racecheck_multirank.log
timeout 900 compute-sanitizer --tool synccheck --print-limit 20 python -m pytest tests/test_gpu_multirank.py tests/test_gpu_compact.py -q -x -p no:cacheprovider -k "two_stream or local_update" > gpurun_out/r2f_synccheck.log 2>&1; echo "synccheck rc=$?"
tail -5 gpurun_out/r2f_synccheck.log
timeout 900 python -m pytest tests/test_gpu_bench_multirank.py -q -x -p no:cacheprovider > gpurun_out/r2f_multirank_bench.log 2>&1; echo "multirank bench rc=$?"
tail -5 gpurun_out/r2f_multirank_bench.log
