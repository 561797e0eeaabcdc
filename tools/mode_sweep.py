"""Time the throughput kernel (mode 1) vs the S-box-split latency kernel (mode 2) vs auto
over launch sizes, to set kSplitMaxTiles (dev aid; prints a table)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2007_10752_b200 as tdes  # noqa: E402
import synthetic  # noqa: E402


def t(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return sorted(ts)[len(ts) // 2]


def main():
    s = tdes.key_schedule(*synthetic.KEYS_3KEY)
    N = 1 << 24
    x = torch.empty(8 * N, dtype=torch.uint8, device="cuda")
    tdes.fill_splitmix64(x)
    y = torch.empty_like(x)
    print("log2n  mode1_ms  mode2_ms  auto_ms  mode1_GBs mode2_GBs auto_GBs")
    for e in range(2, 25):
        n = 1 << e
        xs, ys = x[:8 * n], y[:8 * n]
        r = [t(lambda m=m: tdes.ecb_crypt_mode(xs, s, m, out=ys)) for m in (1, 2, 0)]
        print(f"{e:5d} " + " ".join(f"{v:9.4f}" for v in r) + " " + " ".join(f"{n * 8 / v / 1e6:9.2f}" for v in r),
              flush=True)


if __name__ == "__main__":
    main()
