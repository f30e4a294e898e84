for r in 1 2; do for v in paper_2507_09029_b200/_lib tools/_variants/scatacc; do
  timeout 600 python tools/variant_probe.py $v/libsdp.so s3,s4 >> gpurun_out/ab15.jsonl 2>> gpurun_out/ab15.err
done; done
