# A/B of libsdp source variants (tools/variant_build.py) on one box:
#   python tools/variant_build.py NAME path/to/sdp_sync.cu   (here, per variant)
#   gpurun -- 'bash tools/gpu_r2_variants.sh "A B" c2,c3,c3agg'
for v in $1; do timeout 600 python tools/variant_probe.py tools/_variants/$v/libsdp.so ${2:-c2,c3,c3agg} >> gpurun_out/variants.jsonl 2>> gpurun_out/variants.err; echo "$v rc=$?"; done
