timeout 900 python -m pytest tests/test_gpu_masks.py tests/test_gpu_spec.py -x -q -p no:cacheprovider > gpurun_out/pytest_masks10.log 2>&1; echo "pytest rc=$?"
for r in 1 2; do for v in tools/_variants/head tools/_variants/buildhyb; do
  timeout 600 python tools/variant_probe.py $v/libsdp.so b2,b3,b4 >> gpurun_out/ab10.jsonl 2>> gpurun_out/ab10.err
done; done
