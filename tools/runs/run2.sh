set -x
timeout 600 python tools/l2fetch_probe.py > gpurun_out/l2fetch.jsonl 2> gpurun_out/l2fetch.err; echo "probe rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_owner_sync -s 3 -c 1 \
  -o gpurun_out/c3agg_stream python tools/variant_probe.py paper_2507_09029_b200/_lib/libsdp.so c3agg > gpurun_out/ncu_c3agg.log 2>&1; echo "ncu rc=$?"
