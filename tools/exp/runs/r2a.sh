set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1_smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r1_gputests.log 2>&1
python bench.py > gpurun_out/r1_bench.json 2> gpurun_out/r1_bench.err
python tools/exp/size_timing.py --modes 0,1,2 --lo 14 --hi 24 > gpurun_out/r1_sizes.txt 2>&1
python tools/exp/size_timing.py --modes 0 --lo 25 --hi 27 >> gpurun_out/r1_sizes.txt 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/param_lat tools/exp/param_lat.cu && /tmp/param_lat > gpurun_out/r1_param_lat.txt 2>&1
ncu --metrics smsp__inst_executed_pipe_alu.sum,smsp__inst_executed_pipe_fma.sum,smsp__inst_executed.sum,sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:tdes_ecb_kernel -s 2 -c 1 --csv python tools/profile_kernel.py > gpurun_out/r1_counters.csv 2>&1
tail -3 gpurun_out/r1_gputests.log
cat gpurun_out/r1_bench.json
