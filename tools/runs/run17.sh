timeout 600 python -m pytest tests/test_gpu_sync.py -x -q -p no:cacheprovider -k "stream or direct" > gpurun_out/pytest17_base.log 2>&1
for r in 1 2; do for v in paper_2507_09029_b200/_lib tools/_variants/slot4; do
  timeout 600 python tools/variant_probe.py $v/libsdp.so c3agg,c4nagg,c5n >> gpurun_out/ab17.jsonl 2>> gpurun_out/ab17.err
done; done
