# final refresh at the templated split kernel: smoke, GPU suite, bench, split ncu, sweep, sizes
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin4_smoke.log 2>&1
timeout 2000 python -m pytest tests -m gpu -q > gpurun_out/fin4_gputests.log 2>&1
tail -3 gpurun_out/fin4_gputests.log
python bench.py > gpurun_out/fin4_bench.json 2> gpurun_out/fin4_bench.err
ncu --set full --clock-control none --import-source on -k regex:tdes_split -s 2 -c 1 -o gpurun_out/fin4_prof_split python tools/profile_kernel.py --log2n 17 > /dev/null 2>&1
python tests/helpers/sweep_c2.py --out gpurun_out/fin4_sweep_c2.md > gpurun_out/fin4_sweep.log 2>&1
python tools/exp/size_timing.py --modes 0,1,2,3 --lo 10 --hi 27 > gpurun_out/fin4_sizes.txt 2>&1
cat gpurun_out/fin4_smoke.log | tail -1
cat gpurun_out/fin4_bench.json
