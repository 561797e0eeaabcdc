# last verification pass of the session (HEAD): smoke, GPU suite, bench, reference arm
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin5_smoke.log 2>&1
timeout 2000 python -m pytest tests -m gpu -q > gpurun_out/fin5_gputests.log 2>&1
tail -3 gpurun_out/fin5_gputests.log
python bench.py > gpurun_out/fin5_bench.json 2> gpurun_out/fin5_bench.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/fin5_bench_ref.json 2> gpurun_out/fin5_bench_ref.err
cat gpurun_out/fin5_smoke.log | tail -1
cat gpurun_out/fin5_bench.json
