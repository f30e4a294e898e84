timeout 900 python -m pytest tests/test_gpu_sync.py tests/test_gpu_spec.py tests/test_gpu_fullsize.py -x -q -p no:cacheprovider > gpurun_out/pytest_sync5.log 2>&1; echo "pytest rc=$?"
for r in 1 2; do for v in tools/_variants/head tools/_variants/meanvec paper_2507_09029_b200/_lib tools/_variants/s5; do
  timeout 600 python tools/variant_probe.py $v/libsdp.so c3agg,c4nagg,c5n >> gpurun_out/ab5.jsonl 2>> gpurun_out/ab5.err
done; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_owner_sync -s 3 -c 1 \
  -o gpurun_out/c3agg_stream_mean python tools/variant_probe.py paper_2507_09029_b200/_lib/libsdp.so c3agg > gpurun_out/ncu_c3agg5.log 2>&1; echo "ncu rc=$?"
