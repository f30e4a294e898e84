timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_multirank.py -q -x -p no:cacheprovider -k "two_stream" > gpurun_out/r2y_racecheck_multirank.log 2>&1; echo "racecheck multirank rc=$?"
tail -3 gpurun_out/r2y_racecheck_multirank.log
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_masks.py -q -x -p no:cacheprovider -k "permutation or grouped" > gpurun_out/r2y_racecheck_assign.log 2>&1; echo "racecheck assign rc=$?"
tail -3 gpurun_out/r2y_racecheck_assign.log
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_models.py -q -x -p no:cacheprovider -k "deterministic" > gpurun_out/r2y_racecheck_gn.log 2>&1; echo "racecheck gn rc=$?"
tail -3 gpurun_out/r2y_racecheck_gn.log
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_models.py -q -x -p no:cacheprovider -k "slice_batch or deterministic" > gpurun_out/r2y_memcheck_slices_gn.log 2>&1; echo "memcheck rc=$?"
tail -3 gpurun_out/r2y_memcheck_slices_gn.log
