"""Per-source-line instruction counts / stall samples of one kernel.
usage: python exp/line_prof.py <nvdisasm -g output> <mangled kernel name> <ncu source-page sass csv>"""
import csv, re, sys, collections
dis, kname, sass = sys.argv[1:4]
off2loc, cur, inside = {}, None, False
for line in open(dis):
    if line.startswith("//----") :
        inside = kname in line
        continue
    if not inside: continue
    m = re.search(r'File "([^"]+)", line (\d+)', line)
    if m: cur = (m.group(1).split('/')[-1], int(m.group(2))); continue
    m = re.match(r'\s+/\*([0-9a-f]{4,})\*/\s+(.*)', line)
    if m: off2loc[int(m.group(1), 16)] = (cur, m.group(2).split(';')[0].strip())
rows = list(csv.reader(open(sass)))
hdr = next(r for r in rows if 'Instructions Executed' in r)
hi = rows.index(hdr)
ii, si = hdr.index('Instructions Executed'), hdr.index('Warp Stall Sampling (All Samples)')
base = None
agg = collections.defaultdict(lambda: [0, 0])
opagg = collections.defaultdict(lambda: [0, 0])
for r in rows[hi + 1:]:
    if len(r) < len(hdr) or not r[0].startswith('0x'): continue
    a = int(r[0], 16)
    base = a if base is None else base
    loc, ins = off2loc.get(a - base, (None, r[1]))
    n, s = float(r[ii] or 0), float(r[si] or 0)
    agg[loc][0] += n; agg[loc][1] += s
    op = ins.split()[0] if ins else '?'
    if op.startswith('@'): op = ins.split()[1]
    opagg[op.split('.')[0]][0] += n; opagg[op.split('.')[0]][1] += s
tot = sum(v[0] for v in agg.values()); st = sum(v[1] for v in agg.values())
print(f"total warp-instructions {tot:.4g}, samples {st:.4g}")
src = {}
for loc in agg:
    if loc and loc[0] not in src:
        try: src[loc[0]] = open('paper_2602_22421_b200/csrc/' + loc[0]).read().splitlines()
        except Exception: src[loc[0]] = []
for loc, (n, s) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:int(sys.argv[4]) if len(sys.argv) > 4 else 50]:
    text = src.get(loc[0], [])[loc[1] - 1].strip()[:90] if loc and loc[1] - 1 < len(src.get(loc[0], [])) else ''
    print(f"{n / tot * 100:5.1f}% inst {s / st * 100:5.1f}% samp  {loc[0] if loc else '?'}:{loc[1] if loc else ''}  {text}")
print("by opcode:")
for op, (n, s) in sorted(opagg.items(), key=lambda kv: -kv[1][0])[:25]:
    print(f"  {op:12s} {n / tot * 100:5.1f}% inst {s / st * 100:5.1f}% samp")
