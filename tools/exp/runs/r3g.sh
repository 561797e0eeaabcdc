# circuits: resub S4 18 (same folds), + S2 23 (one fold fewer) vs current; split key-init A/B
set -x
python tools/exp/ab_variants.py tools/exp/v0.so tools/exp/v_s4.so tools/exp/v_s4s2.so tools/exp/v0.so tools/exp/v_s4.so tools/exp/v_s4s2.so > gpurun_out/g_ab_variants.txt 2>&1
python tools/exp/ab_small.py tools/exp/base.so paper_2007_10752_b200/libtdes_b200.so tools/exp/base.so paper_2007_10752_b200/libtdes_b200.so > gpurun_out/g_ab_small.txt 2>&1
TDES_LIB_PATH=tools/exp/strace.so python tools/exp/split_phases.py 1024 16384 131072 > gpurun_out/g_phases.txt 2>&1
cat gpurun_out/g_ab_variants.txt gpurun_out/g_ab_small.txt gpurun_out/g_phases.txt
