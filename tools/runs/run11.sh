for r in 1 2; do for v in paper_2507_09029_b200/_lib tools/_variants/streamwb2; do
  timeout 600 python tools/variant_probe.py $v/libsdp.so c3,c3s,c5n >> gpurun_out/ab11.jsonl 2>> gpurun_out/ab11.err
done; done
