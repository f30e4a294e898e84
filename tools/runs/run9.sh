timeout 900 python -m pytest tests/test_gpu_masks.py -x -q -p no:cacheprovider > gpurun_out/pytest_masks9.log 2>&1; echo "pytest rc=$?"
for r in 1 2; do for v in tools/_variants/head tools/_variants/buildblk tools/_variants/buildgrp; do
  timeout 600 python tools/variant_probe.py $v/libsdp.so b2,b3,b4 >> gpurun_out/ab9.jsonl 2>> gpurun_out/ab9.err
done; done
