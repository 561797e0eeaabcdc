"""Host cost of one call through the Python binding vs the raw C ABI (experiment aid).

Times (wall clock, host side) N back-to-back calls on a tiny input -- the launch is
asynchronous, so this is the host's submission cost per call -- through
tdes.ecb_encrypt (argument checks, device context, stream lookup, ctypes) and through
the C function with every argument precomputed.
"""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_2007_10752_b200 as tdes  # noqa: E402
import synthetic  # noqa: E402

s = tdes.key_schedule(*synthetic.KEYS_3KEY)
for n in (1024, 1 << 17):
    x = torch.empty(8 * n, dtype=torch.uint8, device="cuda"); tdes.fill_splitmix64(x)
    y = torch.empty_like(x)
    N = 2000
    for _ in range(50):
        tdes.ecb_encrypt(x, s, out=y)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(N):
        tdes.ecb_encrypt(x, s, out=y)
    t_py = (time.perf_counter() - t) / N
    torch.cuda.synchronize()
    fn = tdes._lib.tdes_ecb_encrypt
    args = (ctypes.byref(s), x.data_ptr(), y.data_ptr(), n, torch.cuda.current_stream().cuda_stream)
    t = time.perf_counter()
    for _ in range(N):
        fn(*args)
    t_c = (time.perf_counter() - t) / N
    torch.cuda.synchronize()
    # the pieces of the binding
    t = time.perf_counter()
    for _ in range(N):
        torch.cuda.current_stream(x.device).cuda_stream
    t_stream = (time.perf_counter() - t) / N
    t = time.perf_counter()
    for _ in range(N):
        with torch.cuda.device(x.device):
            pass
    t_dev = (time.perf_counter() - t) / N
    print(f"n={n}: binding {t_py * 1e6:.2f} us/call, raw C ABI {t_c * 1e6:.2f} us/call; "
          f"current_stream {t_stream * 1e6:.2f} us, device context {t_dev * 1e6:.2f} us", flush=True)
