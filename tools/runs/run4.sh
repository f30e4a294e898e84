for r in 1 2; do for v in head emitonly predonly meanvec; do
  timeout 600 python tools/variant_probe.py tools/_variants/$v/libsdp.so c3agg,c4nagg,c5n >> gpurun_out/ab4.jsonl 2>> gpurun_out/ab4.err
done; done
