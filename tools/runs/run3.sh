set -x
timeout 900 python -m pytest tests/test_gpu_sync.py tests/test_gpu_spec.py tests/test_gpu_fullsize.py -x -q -p no:cacheprovider > gpurun_out/pytest_sync.log 2>&1; echo "pytest rc=$?"
for lib in tools/_variants/head/libsdp.so paper_2507_09029_b200/_lib/libsdp.so tools/_variants/head/libsdp.so paper_2507_09029_b200/_lib/libsdp.so; do
  timeout 600 python tools/variant_probe.py $lib c3agg,c3,c3s,c4nagg,c4n,c4ns,c5n >> gpurun_out/ab3.jsonl 2>> gpurun_out/ab3.err
done
