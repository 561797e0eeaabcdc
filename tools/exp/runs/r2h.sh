# round 2: measurement pass at T = 182 (GPU suite, bench, reference arm, ncu capture + launch list)
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2h_smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2h_gputests.log 2>&1
tail -3 gpurun_out/r2h_gputests.log
python bench.py > gpurun_out/r2h_bench.json 2> gpurun_out/r2h_bench.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2h_bench_ref.json 2> gpurun_out/r2h_bench_ref.err
ncu --set full --metrics smsp__inst_executed_pipe_alu.sum,smsp__inst_executed_pipe_fma.sum --clock-control none --import-source on -k regex:tdes_ecb_kernel -s 2 -c 1 -o gpurun_out/r2h_prof python tools/profile_kernel.py > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2h_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
cat gpurun_out/r2h_smoke.log | tail -1
cat gpurun_out/r2h_bench.json
