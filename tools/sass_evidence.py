"""Blackwell-native instruction evidence of the built library (CPU box; tooling).

    python tools/sass_evidence.py [lib] > profiles/r02_sass_evidence.md

Counts, per kernel, the SASS mnemonics that only tcgen05 / TMA / bulk-copy / mbarrier code
produces (B200_PROFILING.md "What proves a Blackwell-native kernel"): UTC*MMA (tcgen05.mma),
LDTM / STTM (tcgen05.ld / st), UTCBAR (tcgen05.commit), UBLKCP / UTMALDG (cp.async.bulk[.tensor]),
SYNCS (mbarrier), plus HMMA (legacy mma.sync) to show there is none."""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "paper_1509_08863_b200", "libsc_b200.so")
out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
pat = re.compile(r"\b(UTC[A-Z0-9]*MMA[A-Z0-9.]*|LDTM[A-Z0-9.]*|STTM[A-Z0-9.]*|UTCBAR[A-Z0-9.]*|UBLKCP[A-Z0-9.]*|"
                 r"UTMALDG[A-Z0-9.]*|UTMASTG[A-Z0-9.]*|SYNCS[A-Z0-9.]*|HMMA[A-Z0-9.]*|FFMA2|FADD2)\b")
cnt = collections.defaultdict(collections.Counter)
fn = None
for ln in out.splitlines():
    if "Function :" in ln:
        fn = ln.split("Function :")[1].strip()
        continue
    if fn is None:
        continue
    m = pat.search(ln)
    if m:
        cnt[fn][m.group(1).split(".")[0]] += 1


def short(name):
    m = re.search(r"(\w+?kernel\w*?)(I|E|$)", name)
    return name if not m else name


def demangle(names):
    r = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True)
    return r.stdout.splitlines() if r.returncode == 0 else names


names = sorted(cnt)
dem = demangle(names)
print("# SASS evidence of the Blackwell-native paths (`tools/sass_evidence.py`)\n")
print(f"Library: `{os.path.relpath(lib, ROOT)}` (sm_100a).  Kernels with tcgen05 / TMA / bulk-copy / "
      "mbarrier / packed-fp32 instructions, counts of static SASS instructions per mnemonic:\n")
print("| kernel | mnemonics |")
print("|---|---|")
for n, d in zip(names, dem):
    d = d.replace("(anonymous namespace)::", "").replace("void ", "")
    d = re.sub(r"\(.*", "", d)
    if len(d) > 90:
        d = d[:90] + "…"
    ms = ", ".join(f"{k} {v}" for k, v in sorted(cnt[n].items()))
    print(f"| `{d}` | {ms} |")
hmma = sum(c["HMMA"] for c in cnt.values())
print(f"\nLegacy `HMMA` (mma.sync / wmma) instructions in the whole library: {hmma}.")
