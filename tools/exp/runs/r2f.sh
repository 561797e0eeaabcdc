# round 2: measurement pass at the current build (GPU suite, bench, sweep, ncu, multi-rank launch paths)
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2f_smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2f_gputests.log 2>&1
tail -3 gpurun_out/r2f_gputests.log
python bench.py > gpurun_out/r2f_bench.json 2> gpurun_out/r2f_bench.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2f_bench_ref.json 2> gpurun_out/r2f_bench_ref.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node=1 --master-addr=127.0.0.1 --master-port=29511 bench.py --gpus 1 --steps 10 --no-cpu-baseline > gpurun_out/r2f_bench_torchrun1.json 2> gpurun_out/r2f_bench_torchrun1.err
python bench.py --gpus 2 --steps 3 > gpurun_out/r2f_bench_gpus2.json 2> gpurun_out/r2f_bench_gpus2.err; echo "gpus2 rc=$?" >> gpurun_out/r2f_bench_gpus2.err
ncu --set full --metrics smsp__inst_executed_pipe_alu.sum,smsp__inst_executed_pipe_fma.sum --clock-control none --import-source on -k regex:tdes_ecb_kernel -s 2 -c 1 -o gpurun_out/r2f_prof python tools/profile_kernel.py > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2f_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --metrics smsp__inst_executed_pipe_alu.sum,smsp__inst_executed_pipe_fma.sum --clock-control none --import-source on -k regex:tdes_ecb_kernel -s 2 -c 1 -o gpurun_out/r2f_prof_21 python tools/profile_kernel.py --log2n 21 > /dev/null 2>&1
python tests/helpers/sweep_c2.py --out gpurun_out/r2f_sweep_c2.md > gpurun_out/r2f_sweep.log 2>&1
python tools/exp/size_timing.py --modes 0,1,2,3 --lo 10 --hi 27 > gpurun_out/r2f_sizes.txt 2>&1
cat gpurun_out/r2f_bench.json; cat gpurun_out/r2f_bench_torchrun1.json; tail -2 gpurun_out/r2f_bench_gpus2.err
