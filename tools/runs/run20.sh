for r in 1 2; do for v in paper_2507_09029_b200/_lib tools/_variants/nocheck; do
  timeout 600 python tools/variant_probe.py $v/libsdp.so c3agg,c4nagg,c5n 2>/dev/null | grep aggregate
done; done
