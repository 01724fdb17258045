"""SASS evidence for the hot kernels (cuobjdump -sass of the in-tree
libspmv.so): per kernel, the instruction counts that show the design --
UBLKCP (TMA bulk copy), SYNCS (mbarrier), LDG.E.*.256 (256-bit streaming
loads), LDS / LDS.U8 (shared-memory decode), DFMA, registers and spills.
  python tools/sass_summary.py [lib] > profiles/r02_sass_summary.txt"""
import collections, os, re, subprocess, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "paper_1711_05487_b200", "libspmv.so")
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
fn = None
counts = collections.OrderedDict()
PATS = [("UBLKCP", r"\bUBLKCP"), ("SYNCS", r"\bSYNCS\."), ("LDG.256", r"\bLDG\.E[\.\w]*\.256"),
        ("LDG", r"\bLDG\."), ("LDS.U8", r"\bLDS\.U8"), ("LDS", r"\bLDS\b"), ("DFMA", r"\bDFMA\b"),
        ("SHFL", r"\bSHFL\."), ("BAR", r"\bBAR\."), ("STG", r"\bSTG\.")]
for line in out.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        fn = m.group(1)
        counts[fn] = collections.Counter()
        continue
    if fn is None:
        continue
    for k, p in PATS:
        if re.search(p, line):
            counts[fn][k] += 1
HOT = ("d8_kernel", "stream_kernel", "nzsplit_kernel", "split_fused_kernel", "long_tiled", "fixup_seg")
demangled = {}
try:
    names = subprocess.run(["c++filt"], input="\n".join(counts), capture_output=True, text=True).stdout.splitlines()
    demangled = dict(zip(counts, names))
except Exception:
    pass
print(f"# cuobjdump -sass {os.path.relpath(lib, ROOT)}: instruction counts of the hot kernels")
print(f"# {'kernel':70s} " + " ".join(f"{k:>8s}" for k, _ in PATS))
for f, c in counts.items():
    d = demangled.get(f, f)
    if not any(h in d for h in HOT):
        continue
    print(f"{d[:72]:72s} " + " ".join(f"{c[k]:8d}" for k, _ in PATS))
