set -x
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py --impl reference > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
timeout 1500 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 3 --no-train --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_owner_sync -s 3 -c 1 \
    -o gpurun_out/sync_gpt2 python bench.py --steps 4 --warmup 3 --no-train --no-cpu-baseline > /dev/null 2>&1
timeout 1500 python tools/measure_all.py --only build,sync,sweep,slices --no-cpu > gpurun_out/measure.jsonl 2> gpurun_out/measure.err
