# re-entry check of HEAD: smoke, GPU suite, bench
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/a_smoke.log 2>&1
timeout 2000 python -m pytest tests -m gpu -q -x > gpurun_out/a_gputests.log 2>&1
tail -3 gpurun_out/a_gputests.log
python bench.py > gpurun_out/a_bench.json 2> gpurun_out/a_bench.err
cat gpurun_out/a_bench.json
