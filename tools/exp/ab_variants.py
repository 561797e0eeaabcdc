"""A/B device timing of library builds (experiment aid, not the bench).

Usage: python tools/exp/ab_variants.py a.so b.so ... [--rounds 2]
Each build runs in its own process (TDES_LIB_PATH) on the bench workload
(1 GiB 3DES encrypt, 3-key) and prints the median launch time; variants are
interleaved `rounds` times.  The ciphertext sum64 must agree across builds.
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
n = 1 << 27
x = torch.empty(8 * n, dtype=torch.uint8, device="cuda"); tdes.fill_splitmix64(x)
y = torch.empty_like(x)
s = tdes.key_schedule(*synthetic.KEYS_3KEY)
res = {}
ds = tdes.des_key_schedule(synthetic.KEYS_1KEY[0])
for name, fn in (("enc", lambda: tdes.ecb_encrypt(x, s, out=y)), ("des", lambda: tdes.des_ecb_encrypt(x, ds, out=y))):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(20):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); b.synchronize(); ts.append(a.elapsed_time(b))
    ts.sort()
    res[name] = ts[len(ts) // 2]
tdes.ecb_encrypt(x, s, out=y)
d = tdes.sum64(y)
tdes.des_ecb_encrypt(x, ds, out=y)
d2 = tdes.sum64(y)
print(f"RESULT enc_ms={res['enc']:.4f} GBps={n*8/res['enc']/1e6:.1f} sum64={d:016x} des_GBps={n*8/res['des']/1e6:.1f} des_sum64={d2:016x}")
'''.replace("ROOT", repr(ROOT))


def main():
    args = sys.argv[1:]
    rounds = 2
    if "--rounds" in args:
        i = args.index("--rounds")
        rounds = int(args[i + 1])
        del args[i:i + 2]
    for r in range(rounds):
        for so in args:
            env = dict(os.environ, TDES_LIB_PATH=os.path.abspath(so))
            out = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
            line = [ln for ln in out.stdout.splitlines() if ln.startswith("RESULT")]
            print(f"round {r} {os.path.basename(so)}: {line[0] if line else out.stderr[-800:]}", flush=True)


if __name__ == "__main__":
    main()
