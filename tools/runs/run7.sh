timeout 900 python -m pytest tests/test_gpu_sync.py tests/test_gpu_spec.py tests/test_gpu_fullsize.py -x -q -p no:cacheprovider > gpurun_out/pytest_sync7.log 2>&1; echo "pytest rc=$?"
for r in 1 2; do for v in tools/_variants/head paper_2507_09029_b200/_lib tools/_variants/meanpred; do
  timeout 600 python tools/variant_probe.py $v/libsdp.so c3agg,c4nagg,c5n >> gpurun_out/ab7.jsonl 2>> gpurun_out/ab7.err
done; done
