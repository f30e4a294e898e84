# Reproduce the round's GPU evidence on one B200 (run under gpurun; outputs in gpurun_out/):
#   gpurun --timeout 5400 -- 'bash tools/gpu_evidence.sh'
set -x
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py --impl reference > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
timeout 1500 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
# launch list of the bench command (per-launch times are cold and serialised: compare shares)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 3 --no-train --no-cpu-baseline > /dev/null 2>&1
# the headline kernel, full set (DRAM bytes -> profiles/traffic.json)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_owner_sync -s 3 -c 1 \
    -o gpurun_out/sync_gpt2 python bench.py --steps 4 --warmup 3 --no-train --no-cpu-baseline > /dev/null 2>&1
timeout 1500 python tools/measure_all.py --only build,sync,sweep,slices --no-cpu > gpurun_out/measure.jsonl 2> gpurun_out/measure.err
timeout 700 python tools/small_probe.py --sizes 1,4,16,64 --ps 2,4,8 > gpurun_out/small.jsonl 2> gpurun_out/small.err
timeout 900 python tools/equal_loss.py --steps 1500 --out gpurun_out/equal_loss.json > /dev/null 2>&1
timeout 900 compute-sanitizer --tool racecheck python -m pytest tests/test_gpu_multirank.py -q -x -p no:cacheprovider \
    -k two_stream > gpurun_out/racecheck_multirank.log 2>&1
