"""Build tools/exp/strace.so: the product library with a per-round clock64 trace of
the split kernel's CTA 0 (arrival at / release from each round's barrier, per warp),
read by tools/exp/split_trace.py (experiment aid).

  python tools/exp/split_trace_build.py [--out tools/exp/strace.so] [-D X=1 ...]
"""
import argparse
import os
import shutil
import subprocess
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

GLOBALS = r'''
__device__ long long g_strace[8][2][100];
__device__ unsigned long long g_sphase[8][6];    // CTA 0, per warp: entry, keys, loaded, rounds, stored, exit
__device__ unsigned long long g_scta[1024][2];   // per CTA (warp 0): entry, exit
__device__ __forceinline__ unsigned long long gt_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
'''


def patch(t: str) -> str:
    t = t.replace("namespace {\n", "namespace {\n" + GLOBALS, 1)
    head = "  const size_t ntiles = (nblocks + kGroupBlocks - 1) / kGroupBlocks;\n"
    assert head in t
    t = t.replace(head, "  long long* tr = (blockIdx.x == 0 && lane == 0) ? &g_strace[G][0][0] : nullptr;\n  int ri = 0;\n" + head, 1)
    rhead = "  const int G = GC >= 0 ? GC : G_;"
    assert rhead in t
    t = t.replace(rhead, rhead + "\n  long long* tr = (blockIdx.x == 0 && lane == 0) ? &g_strace[G][0][0] : nullptr;\n  int ri = 0;", 1)
    for old in ("      split_keys(ks, r + 1, c, S, K);\n      team_sync<WPT>();\n",
                "      if (r + 2 < 16 * NSTAGES) split_keys(ks, r + 2, c, S, K);\n      team_sync<WPT>();\n"):
        assert old in t, old
        new = old.replace("      team_sync<WPT>();\n",
                          "      if (tr && ri < 100) tr[ri] = clock64();\n      team_sync<WPT>();\n"
                          "      if (tr && ri < 100) tr[100 + ri] = clock64();\n      ++ri;\n")
        t = t.replace(old, new, 1)
    ph = [("  const unsigned lane = threadIdx.x & 31u;\n  const int g = threadIdx.x >> 5;  // this warp\n",
           "  const bool ph0 = blockIdx.x == 0 && lane == 0;\n  if (ph0) g_sphase[g][0] = gt_now();\n"
           "  if (lane == 0 && g == 0 && blockIdx.x < 1024) g_scta[blockIdx.x][0] = gt_now();\n"),
          ("  __syncwarp();\n  split_body<WPT, NSTAGES, SPEC>(", ""),
          ("    if (SPEC) {\n      split_rounds_spec", "PREFIX    if (tr && tile == blockIdx.x) g_sphase[G][2] = gt_now();\n"),
          ("    // FP (renaming) + store: warp G writes the groups it loaded\n", "    if (tr && tile == blockIdx.x) g_sphase[G][3] = gt_now();\n"),
          ("    team_sync<WPT>();\n  }\n}\n", "    if (tr && tile == blockIdx.x) g_sphase[G][4] = gt_now();\n")]
    for anchor, ins in ph:
        assert anchor in t, anchor
        if anchor.startswith("  __syncwarp();\n  split_body"):
            t = t.replace(anchor, "  __syncwarp();\n  if (ph0) g_sphase[g][1] = gt_now();\n  split_body<WPT, NSTAGES, SPEC>(", 1)
        elif ins.startswith("PREFIX"):
            t = t.replace(anchor, ins[len("PREFIX"):] + anchor, 1)
        else:
            t = t.replace(anchor, anchor + ins if not anchor.startswith("    team_sync") else ins + anchor, 1)
    tail = "  split_body<WPT, NSTAGES, SPEC>(g, in, out, nblocks, st, ks.r[g], lane, c);\n}\n"
    assert tail in t
    t = t.replace(tail, tail[:-2] + "  if (ph0) g_sphase[g][5] = gt_now();\n"
                  "  if (lane == 0 && g == 0 && blockIdx.x < 1024) g_scta[blockIdx.x][1] = gt_now();\n}\n", 1)
    return t + '''
extern "C" int tdes_get_sphase(void* host, void* cta) {
  if (cudaMemcpyFromSymbol(host, g_sphase, sizeof g_sphase) != cudaSuccess) return TDES_ERR_CUDA;
  return cudaMemcpyFromSymbol(cta, g_scta, sizeof g_scta) == cudaSuccess ? 0 : TDES_ERR_CUDA;
}
extern "C" int tdes_get_strace(void* host) {
  return cudaMemcpyFromSymbol(host, g_strace, sizeof g_strace) == cudaSuccess ? 0 : TDES_ERR_CUDA;
}
'''


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(HERE, "strace.so"))
    ap.add_argument("-D", dest="define", action="append", default=[], type=lambda v: "-D" + v)
    a = ap.parse_args()
    import __graft_entry__ as ge
    tmp = tempfile.mkdtemp(prefix="tdes_strace_")
    shutil.copytree(ge.CSRC, os.path.join(tmp, "pkg", "csrc"))
    shutil.copytree(os.path.join(ROOT, "include"), os.path.join(tmp, "include"))
    src = os.path.join(tmp, "pkg", "csrc")
    k = os.path.join(src, "tdes_kernel.cu")
    text = open(k).read()
    open(k, "w").write(patch(text))
    cmd = [ge._nvcc(), *ge.NVCC_FLAGS, *a.define, "-o", os.path.abspath(a.out), *[os.path.join(src, s) for s in ge.SOURCES]]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode:
        sys.exit(r.stderr[-3000:])
    print("built", a.out)


if __name__ == "__main__":
    main()
