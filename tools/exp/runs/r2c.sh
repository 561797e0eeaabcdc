# round 2: GPU suite with the auto devkeys window; ncu of mid sizes; c4/c5 bench lines at N=1
set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2c_gputests.log 2>&1
tail -3 gpurun_out/r2c_gputests.log
for m in 1 3; do
  ncu --set full --clock-control none --import-source on -k regex:tdes_ecb_kernel -s 2 -c 1 -o gpurun_out/r2c_prof_19_m$m python tools/profile_kernel.py --log2n 19 --mode $m > /dev/null 2>&1
done
ncu --set full --clock-control none --import-source on -k regex:tdes_ecb_kernel -s 2 -c 1 -o gpurun_out/r2c_prof_21_m1 python tools/profile_kernel.py --log2n 21 --mode 1 > /dev/null 2>&1
python tools/exp/size_timing.py --modes 0 --lo 14 --hi 27 > gpurun_out/r2c_sizes_auto.txt 2>&1
python bench.py --workload c4 --steps 10 --no-cpu-baseline > gpurun_out/r2c_bench_c4.json 2> gpurun_out/r2c_bench_c4.err
python bench.py --workload c5 --steps 3 --no-cpu-baseline > gpurun_out/r2c_bench_c5.json 2> gpurun_out/r2c_bench_c5.err
cat gpurun_out/r2c_sizes_auto.txt
python -c "
import json
for w in ('c4','c5'):
    d=json.load(open('gpurun_out/r2c_bench_%s.json'%w)); print(w, d['value'], d['check'])"
