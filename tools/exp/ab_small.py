"""A/B of small-launch latency across library builds (experiment aid, not the bench).

Usage: python tools/exp/ab_small.py a.so b.so ...
Per build (own process, TDES_LIB_PATH): for each size, the median device time of
one 3DES encrypt launch (CUDA events), the time per launch of 200 back-to-back
launches, and the output sum64 (must agree across builds).
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
for e in (2, 10, 14, 17, 18, 19, 20):
    n = 1 << e
    x = torch.empty(8 * n, dtype=torch.uint8, device="cuda"); tdes.fill_splitmix64(x)
    y = torch.empty_like(x)
    fn = lambda: tdes.ecb_encrypt(x, s, out=y)
    for _ in range(5): fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(30):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); b.synchronize(); ts.append(a.elapsed_time(b))
    ts.sort()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(200): fn()
    b.record(); b.synchronize()
    per = a.elapsed_time(b) / 200
    fn(); d = tdes.sum64(y)
    print(f"RESULT 2^{e:<2d} single {ts[len(ts)//2]*1e3:8.1f} us  back-to-back {per*1e3:8.1f} us/launch  {n*8/per/1e6:8.1f} GB/s  sum64={d:016x}")
'''.replace("ROOT", repr(ROOT))


def main():
    for so in sys.argv[1:]:
        env = dict(os.environ, TDES_LIB_PATH=os.path.abspath(so))
        out = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
        print(f"== {os.path.basename(so)}")
        lines = [ln[7:] for ln in out.stdout.splitlines() if ln.startswith("RESULT")]
        print("\n".join(lines) if lines else out.stderr[-1500:], flush=True)


if __name__ == "__main__":
    main()
