timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r2e_pytest_gpu.log 2>&1; echo "all rc=$?"
tail -15 gpurun_out/r2e_pytest_gpu.log
timeout 1300 python -c "
import sys, json, argparse; sys.path.insert(0, '.')
import bench
args = argparse.Namespace(p=4, train_steps=6)
print(json.dumps(bench.run_memory_ranks(args)))
" > gpurun_out/r2e_mem.json 2> gpurun_out/r2e_mem.err; echo "rc=$?"
head -c 4000 gpurun_out/r2e_mem.json; tail -20 gpurun_out/r2e_mem.err
