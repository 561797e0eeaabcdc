"""Back-to-back and queued time of launches at tile counts between the powers of two
(experiment aid): python tools/exp/split_tiles.py [--mode 2] [tiles ...]
(mode 2 = the split kernel forced, 1 = the throughput kernel, 0 = auto)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402
import paper_2007_10752_b200 as tdes  # noqa: E402
import synthetic  # noqa: E402

s = tdes.key_schedule(*synthetic.KEYS_3KEY)
args = sys.argv[1:]
mode = 2
if args[:1] == ["--mode"]:
    mode, args = int(args[1]), args[2:]
for t in [int(a) for a in args] or [1, 16, 64, 96, 128, 148, 160, 192, 224, 256, 296]:
    n = t * 1024
    x = torch.empty(8 * n, dtype=torch.uint8, device="cuda"); tdes.fill_splitmix64(x)
    y = torch.empty_like(x)
    fn = lambda: tdes.ecb_crypt_mode(x, s, mode, out=y)
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    q = []
    for _ in range(15):
        torch.cuda._sleep(300_000)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); b.synchronize(); q.append(a.elapsed_time(b))
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(50):
        fn()
    b.record(); b.synchronize()
    print(f"mode {mode} tiles {t:4d}: queued {sorted(q)[7] * 1e3:6.1f} us, back-to-back {a.elapsed_time(b) / 50 * 1e3:6.1f} us, sum64={tdes.sum64(y):016x}", flush=True)
