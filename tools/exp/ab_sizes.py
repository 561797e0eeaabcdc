"""Throughput-kernel time per launch over sizes 2^19..2^27 for several builds (experiment aid).

python tools/exp/ab_sizes.py a.so b.so ...
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
    reps = max(5, min(50, (1 << 31) >> (e + 3)))
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): fn()
    b.record(); b.synchronize()
    out.append(f"{a.elapsed_time(b) / reps * 1e3:9.1f}")
tdes.ecb_crypt_mode(x, s, 1, out=y)
print("RESULT", " ".join(out), f"sum64={tdes.sum64(y):016x}")
'''.replace("ROOT", repr(ROOT))

print("build      " + " ".join(f"{'2^%d' % e:>9s}" for e in range(19, 28)) + "   (us per launch, back-to-back)")
for so in sys.argv[1:]:
    env = dict(os.environ, TDES_LIB_PATH=os.path.abspath(so))
    r = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
    line = [ln for ln in r.stdout.splitlines() if ln.startswith("RESULT")]
    print(f"{os.path.basename(so):10s} " + (line[0][7:] if line else r.stderr[-600:]), flush=True)
