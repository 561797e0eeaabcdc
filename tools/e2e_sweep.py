"""Host-pipeline (tdes_ecb_crypt_host) throughput vs chunk size and stream count (dev aid)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2007_10752_b200 as tdes  # noqa: E402
import synthetic  # noqa: E402


def main():
    n = 1 << 27
    s = tdes.key_schedule(*synthetic.KEYS_3KEY)
    hin = torch.empty(8 * n, dtype=torch.uint8).pin_memory()
    hout = torch.empty_like(hin).pin_memory()
    # plain copy references
    d = torch.empty(8 * n, dtype=torch.uint8, device="cuda")
    for name, fn in (("H2D only", lambda: d.copy_(hin, non_blocking=True)),
                     ("D2H only", lambda: hout.copy_(d, non_blocking=True))):
        fn(); torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); b.synchronize()
        print(f"{name}: {8 * n / a.elapsed_time(b) / 1e6:.1f} GB/s")
    del d
    for chunk_log2 in (19, 20, 21, 22, 23):
        for ns in (2, 3, 4, 6):
            pipe = tdes.HostPipeline(chunk_blocks=1 << chunk_log2, nstreams=ns)
            pipe.run(s, hin, hout)
            torch.cuda.synchronize()
            cur = torch.cuda.current_stream()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(cur)
            for _ in range(3):
                pipe.run(s, hin, hout)
            for st in pipe.streams:
                cur.wait_stream(st)
            b.record(cur); b.synchronize()
            print(f"chunk 2^{chunk_log2} blocks ({(8 << chunk_log2) >> 20} MiB) x {ns} streams: "
                  f"{3 * 8 * n / a.elapsed_time(b) / 1e6:.1f} GB/s", flush=True)
            del pipe


if __name__ == "__main__":
    main()
