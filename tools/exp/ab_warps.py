"""Throughput-kernel time vs warps per CTA and size (experiment aid).

python tools/exp/ab_warps.py tools/exp/wenv.so   (a -DTDES_EXP_WARPS_ENV build)
"""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
CHILD = r'''
import sys, torch
sys.path.insert(0, ROOT)
import paper_2007_10752_b200 as tdes, synthetic
s = tdes.key_schedule(*synthetic.KEYS_3KEY)
x = torch.empty(8 << 27, dtype=torch.uint8, device="cuda"); tdes.fill_splitmix64(x)
y = torch.empty_like(x)
out = []
for e in range(19, 28):
    n = 1 << e
    xs, ys = x[:8 * n], y[:8 * n]
    fn = lambda: tdes.ecb_crypt_mode(xs, s, 1, out=ys)
    for _ in range(3): fn()
    reps = max(3, min(50, (1 << 30) >> (e + 3)))
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): fn()
    b.record(); b.synchronize()
    out.append(f"{a.elapsed_time(b) / reps * 1e3:9.1f}")
print("RESULT", " ".join(out))
'''.replace("ROOT", repr(ROOT))

so = os.path.abspath(sys.argv[1])
print("warps " + " ".join(f"{'2^%d' % e:>9s}" for e in range(19, 28)) + "   (us per launch, back-to-back)")
for w in (8, 9, 10, 11, 12, 13, 14, 15, 16):
    env = dict(os.environ, TDES_LIB_PATH=so, TDES_EXP_WARPS=str(w))
    r = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
    line = [ln for ln in r.stdout.splitlines() if ln.startswith("RESULT")]
    print(f"{w:5d} " + (line[0][7:] if line else r.stderr[-500:]), flush=True)
