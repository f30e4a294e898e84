for r in 1 2; do for v in paper_2507_09029_b200/_lib tools/_variants/gatherpf; do
  timeout 600 python tools/variant_probe.py $v/libsdp.so s3,s4 >> gpurun_out/ab18.jsonl 2>> gpurun_out/ab18.err
done; done
