timeout 1500 python -m pytest tests/test_gpu_models.py tests/test_gpu_layout.py tests/test_gpu_train.py tests/test_gpu_ipc.py -x -q -p no:cacheprovider > gpurun_out/r2q_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r2q_pytest.log
timeout 900 python tools/measure_all.py --only slices > gpurun_out/r2q_slices.jsonl 2> gpurun_out/r2q_slices.err; echo "measure rc=$?"
tail -3 gpurun_out/r2q_slices.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_gather|k_scatter" -s 12 -c 4 -o gpurun_out/r2q_slices python tools/ncu_targets.py slices_all_r18 > gpurun_out/r2q_ncu.log 2>&1; echo "ncu rc=$?"
