# round 2: ncu of the team kernels at 2^19 blocks
set -x
for m in 4 6 5; do
  ncu --set full --clock-control none --import-source on -k regex:tdes_team_kernel -s 2 -c 1 -o gpurun_out/r2e_prof_19_m$m python tools/profile_kernel.py --log2n 19 --mode $m > /dev/null 2>&1
done
ls -la gpurun_out/
