# final measurement pass of the re-entered round-2 session (the committed build)
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin_smoke.log 2>&1
timeout 2000 python -m pytest tests -m gpu -q > gpurun_out/fin_gputests.log 2>&1
tail -3 gpurun_out/fin_gputests.log
python bench.py > gpurun_out/fin_bench.json 2> gpurun_out/fin_bench.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/fin_bench_ref.json 2> gpurun_out/fin_bench_ref.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node=1 --master-addr=127.0.0.1 --master-port=29517 bench.py --gpus 1 --steps 20 --no-cpu-baseline > gpurun_out/fin_bench_torchrun1.json 2> gpurun_out/fin_bench_torchrun1.err
python bench.py --workload c4 --steps 10 --no-cpu-baseline > gpurun_out/fin_bench_c4.json 2> gpurun_out/fin_bench_c4.err
python bench.py --workload c5 --steps 3 --no-cpu-baseline > gpurun_out/fin_bench_c5.json 2> gpurun_out/fin_bench_c5.err
ncu --set full --metrics smsp__inst_executed_pipe_alu.sum,smsp__inst_executed_pipe_fma.sum --clock-control none --import-source on -k regex:tdes_ecb_kernel -s 2 -c 1 -o gpurun_out/fin_prof python tools/profile_kernel.py > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/fin_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --metrics smsp__inst_executed_pipe_alu.sum,smsp__inst_executed_pipe_fma.sum --clock-control none --import-source on -k regex:tdes_ecb_kernel -s 2 -c 1 -o gpurun_out/fin_prof_21 python tools/profile_kernel.py --log2n 21 > /dev/null 2>&1
ncu --set full --metrics smsp__inst_executed_pipe_alu.sum,smsp__inst_executed_pipe_fma.sum --clock-control none --import-source on -k regex:tdes_ecb_kernel -s 2 -c 1 -o gpurun_out/fin_prof_c3 python tools/profile_kernel.py --log2n 25 --keys 2key > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:tdes_ecb_kernel -s 2 -c 1 -o gpurun_out/fin_prof_des python tools/profile_kernel.py --op des > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:tdes_split -s 2 -c 1 -o gpurun_out/fin_prof_split python tools/profile_kernel.py --log2n 17 > /dev/null 2>&1
python tests/helpers/sweep_c2.py --out gpurun_out/fin_sweep_c2.md > gpurun_out/fin_sweep.log 2>&1
python tools/exp/size_timing.py --modes 0,1,2,3 --lo 10 --hi 27 > gpurun_out/fin_sizes.txt 2>&1
cat gpurun_out/fin_smoke.log | tail -1
cat gpurun_out/fin_bench.json
ls -la gpurun_out/
