import csv, re, sys, collections
sass, csvf, upd = sys.argv[1], sys.argv[2], float(sys.argv[3])
addr2line = {}
cur = None
for ln in open(sass):
    m = re.match(r'\s*//## File "([^"]+)", line (\d+)', ln)
    if m:
        cur = (m.group(1).split('/')[-1], int(m.group(2)))
        continue
    m = re.match(r'\s*/\*([0-9a-f]{4,})\*/', ln)
    if m:
        addr2line[int(m.group(1), 16)] = cur
rows = list(csv.reader(open(csvf)))
hdr = rows[1]; ix = {h: i for i, h in enumerate(hdr)}
def f(r, k):
    try: return float(r[ix[k]] or 0)
    except: return 0.0
agg = collections.defaultdict(lambda: [0.0]*5)
base = int(rows[2][ix["Address"]], 16)
tot = sum(f(r, 'Warp Stall Sampling (All Samples)') for r in rows[2:])
for r in rows[2:]:
    a = int(r[ix["Address"]], 16) - base
    key = addr2line.get(a, ('?', 0))
    g = agg[key]
    g[0] += f(r, 'Instructions Executed'); g[1] += f(r, 'L1 Wavefronts Shared'); g[2] += f(r, 'L1 Tag Requests Global')
    g[3] += f(r, 'Warp Stall Sampling (All Samples)')
src = {}
for key in agg:
    pass
lines = open(sys.argv[5] if len(sys.argv) > 5 else '/root/repo/paper_1911_09278_b200/csrc/k_sv.cuh').read().split('\n')
for key, g in sorted(agg.items(), key=lambda x: -x[1][0])[:int(sys.argv[4]) if len(sys.argv) > 4 else 50]:
    s = lines[key[1]-1].strip()[:80] if key[0] == 'k_sv.cuh' else ''
    print('%-22s i/u %6.2f shwf/u %5.2f gtag/u %5.2f stall%% %5.1f | %s' % ('%s:%d' % key, g[0]/upd, g[1]/upd, g[2]/upd, 100*g[3]/tot, s))
