timeout 600 python -m pytest tests/test_gpu_sync.py tests/test_gpu_spec.py -x -q -p no:cacheprovider > gpurun_out/pytest19.log 2>&1; tail -1 gpurun_out/pytest19.log
for r in 1 2; do
timeout 300 python tools/direct_probe.py --aggregate --lib tools/_variants/preleak/libsdp.so 2>&1 | grep cfg
timeout 300 python tools/direct_probe.py --aggregate 2>&1 | grep cfg
done
for v in tools/_variants/preleak paper_2507_09029_b200/_lib; do timeout 600 python tools/variant_probe.py $v/libsdp.so c3agg,c4nagg,c5n 2>/dev/null; done
