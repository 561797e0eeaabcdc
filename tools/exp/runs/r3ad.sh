# box-to-box variance of the size timing (auto mode): run on separate boxes
set -x
nvidia-smi --query-gpu=name,pci.bus_id,clocks.sm,clocks.max.sm --format=csv > gpurun_out/var_$1.txt
python tools/exp/size_timing.py --modes 0 --lo 10 --hi 27 >> gpurun_out/var_$1.txt 2>&1
cat gpurun_out/var_$1.txt
