"""Attribute ncu per-SASS-instruction stall samples / instruction counts to CUDA source lines.

    python tools/ncu_lines.py REPORT.ncu-rep KERNEL_MANGLED_NAME [top]
Needs the .so built with -lineinfo (it is) and nvdisasm; maps SASS offsets to `//## File ... line N`
annotations from `nvdisasm -g`."""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile

rep, fn = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
extra = sys.argv[4] if len(sys.argv) > 4 else "L1 Wavefronts Shared"  # third column, summed per line
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
so = os.path.join(ROOT, "paper_1911_09278_b200", "libmace_b200.so")
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", so], cwd=tmp, capture_output=True)
dis = ""
for cub in sorted(f for f in os.listdir(tmp) if f.endswith(".cubin")):
    d = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(tmp, cub)], capture_output=True, text=True).stdout
    if fn in d:
        dis = d
        break
# walk the function's text
lines = dis.splitlines()
start = next(i for i, l in enumerate(lines) if re.match(r"^\S*" + re.escape(fn) + r"\S*:$", l))
off2line = {}
cur = None
for l in lines[start + 1:]:
    if l.startswith("//---") or (l.startswith(".text.") and fn not in l):
        break
    m = re.search(r'line (\d+)', l)
    if "//##" in l and m:
        cur = int(m.group(1))
        fm = re.search(r'File "([^"]+)"', l)
        cur = (os.path.basename(fm.group(1)) if fm else "?", cur)
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", l)
    if m:
        off2line[int(m.group(1), 16)] = cur
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
h = rows[1]
A, S, I, SRC = h.index("Address"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed"), h.index("Source")
X = h.index(extra) if extra in h else None
base = None
agg_s, agg_i, agg_x = collections.Counter(), collections.Counter(), collections.Counter()
for r in rows[2:]:
    try:
        addr = int(r[A], 16)
    except ValueError:
        continue
    if base is None:
        base = addr
    key = off2line.get(addr - base, ("?", -1))
    agg_s[key] += float(r[S] or 0)
    agg_i[key] += float(r[I] or 0)
    if X is not None:
        agg_x[key] += float(r[X] or 0)
ts, ti, tx = sum(agg_s.values()), sum(agg_i.values()), max(sum(agg_x.values()), 1.0)
srcfiles = {}
def text(f, n):
    p = os.path.join(ROOT, "paper_1911_09278_b200", "csrc", f)
    if f not in srcfiles:
        srcfiles[f] = open(p).read().splitlines() if os.path.exists(p) else []
    L = srcfiles[f]
    return L[n - 1].strip()[:90] if 0 < n <= len(L) else ""
for k, v in agg_s.most_common(top):
    print(f"{v / ts * 100:5.1f}% stall {agg_i[k] / ti * 100:5.1f}% inst {agg_x[k] / tx * 100:5.1f}% x  "
          f"{k[0]}:{k[1]:<4} {text(*k)}")
print(f"total {extra}: {tx:.4g}")
