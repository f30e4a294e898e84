for i in 1 2; do
  python tools/sync_ab.py tools/ab/libsdp_r2a.so gpt2 60
  python tools/sync_ab.py default gpt2 60
done
python tools/sync_ab.py tools/ab/libsdp_r2a.so resnet18 200
python tools/sync_ab.py default resnet18 200
python tools/sync_ab.py tools/ab/libsdp_r2a.so sweep:256 60
python tools/sync_ab.py default sweep:256 60
timeout 600 python -m pytest tests/test_gpu_compact.py tests/test_gpu_sync.py tests/test_gpu_fullsize.py -x -q -p no:cacheprovider 2>&1 | tail -3
