"""Development aid: attribute the SASS a kernel executed (from an ncu
`--page source --csv --print-source sass` export) to source lines, using
`nvdisasm -g` line info of the same cubin.

  python tools/sass_regions.py <ncu_sass.csv> <nvdisasm_-g.sass> <kernel symbol>
"""
import collections
import csv
import re
import sys

csv_path, sass_path, sym = sys.argv[1:4]
rows = list(csv.reader(open(csv_path)))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
base = None
executed = {}
stall = {}
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
stall_by = {}
for r in rows[2:]:
    try:
        a = int(r[0], 16)
        ie = int(r[ix["Instructions Executed"]])
    except Exception:
        continue
    if base is None:
        base = a
    off = a - base
    executed[off] = ie
    stall[off] = int(r[ix["stall_no_inst"]]) if "stall_no_inst" in ix else 0
    stall_by[off] = {c: int(r[ix[c]]) for c in stall_cols}

# line info: walk the kernel's section
lines = open(sass_path).read().split("\n")
start = next(k for k, l in enumerate(lines) if l.startswith(sym + ":"))
cur = None
off2src = {}
for l in lines[start + 1:]:
    if l.startswith("\t.section") or (l and not l[0].isspace() and l.endswith(":") and not l.startswith(".")):
        if off2src:
            break
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", l)
    if m:
        off2src[int(m.group(1), 16)] = cur
by_file_line = collections.Counter()
lines128 = collections.defaultdict(set)
for off, ie in executed.items():
    if ie <= 0:
        continue
    src = off2src.get(off)
    by_file_line[src] += 16
    lines128[src].add(off // 128)
tot = sum(by_file_line.values())
print(f"executed code {tot} B, {len(set(o // 128 for o, e in executed.items() if e > 0))} distinct 128-B lines")
by_file = collections.Counter()
for (src, b) in by_file_line.items():
    by_file[src[0] if src else None] += b
print("by file:", by_file.most_common())
agg = collections.Counter()
for src, b in by_file_line.items():
    if src:
        agg[(src[0], src[1] // 10 * 10)] += b
print("top source regions (file, line//10*10): bytes executed")
for (f, l), b in agg.most_common(40):
    print(f"  {f}:{l:5d}  {b}")

# warp-state samples by source region and reason
tot_s = collections.Counter()
reg_s = collections.defaultdict(collections.Counter)
for off, st in stall_by.items():
    src = off2src.get(off)
    key = (src[0], src[1]) if src else ("?", 0)
    for c, v in st.items():
        if v:
            tot_s[c] += v
            reg_s[key][c] += v
N = sum(tot_s.values())
print(f"samples {N}:", ", ".join(f"{c[6:]} {v * 100 / max(N, 1):.1f}%" for c, v in tot_s.most_common(8)))
print("top source lines by samples:")
for key, cnt in sorted(reg_s.items(), key=lambda kv: -sum(kv[1].values()))[:45]:
    t = sum(cnt.values())
    print(f"  {key[0]}:{key[1]:5d} {t:6d} ({t * 100 / max(N, 1):4.1f}%) " +
          ", ".join(f"{c[6:]} {v}" for c, v in cnt.most_common(3)))
