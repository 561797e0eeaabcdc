# round 2: team kernels (modes 4-7): parity + size timing against modes 1 and 3
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "modes or random_keys or weak" > gpurun_out/r2d_parity.log 2>&1
tail -3 gpurun_out/r2d_parity.log
python tools/exp/size_timing.py --modes 1,3,4,5,6,7 --lo 14 --hi 23 > gpurun_out/r2d_sizes.txt 2>&1
cat gpurun_out/r2d_sizes.txt
