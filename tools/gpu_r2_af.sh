timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2af_pytest.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/r2af_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2af_smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py --impl reference > gpurun_out/r2af_ref.json 2> gpurun_out/r2af_ref.err; echo "ref rc=$?"
timeout 1500 python bench.py > gpurun_out/r2af_bench.json 2> gpurun_out/r2af_bench.err; echo "bench rc=$?"
tail -c 300 gpurun_out/r2af_bench.err
