for r in 1 2; do for v in tools/_variants/head paper_2507_09029_b200/_lib tools/_variants/buildblk; do
  timeout 600 python tools/variant_probe.py $v/libsdp.so b2,b3,b4 >> gpurun_out/ab8.jsonl 2>> gpurun_out/ab8.err
done; done
