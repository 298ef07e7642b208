"""Attribute ncu warp-stall samples of one kernel to CUDA source lines (and stall reasons).

usage: python tools/stall_by_line.py REP.ncu-rep OBJ.o KERNEL_SUBSTR [top]

ncu's SASS page gives per-instruction stall samples at absolute addresses; the same cubin,
disassembled here with `nvdisasm --print-line-info`, maps function-relative offsets to lines.
"""
import collections, csv, io, re, subprocess, sys, tempfile, os

rep, obj, ksub = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 30

src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr = rows[1]
ia, iS = hdr.index("Address"), hdr.index("Warp Stall Sampling (All Samples)")
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
data = [r for r in rows[2:] if len(r) == len(hdr)]
base = int(data[0][ia], 16)

with tempfile.TemporaryDirectory() as td:
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=td, capture_output=True)
    cubins = [f for f in os.listdir(td) if f.endswith(".cubin")]
    lines = {}
    for cb in cubins:
        dis = subprocess.run(["nvdisasm", "--print-line-info", "-c", os.path.join(td, cb)],
                             capture_output=True, text=True).stdout
        fn, cur = None, None
        for ln in dis.splitlines():
            m = re.match(r"\s*\.text\.(\S+):", ln)
            if m:
                fn = m.group(1)
                continue
            m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
            if m:
                cur = (os.path.basename(m.group(1)), int(m.group(2)))
                continue
            m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
            if m and fn and ksub in fn:
                lines[int(m.group(1), 16)] = cur
agg = collections.defaultdict(lambda: collections.Counter())
tot = collections.Counter()
for r in data:
    off = int(r[ia], 16) - base
    key = lines.get(off, ("?", 0))
    s = int(r[iS] or 0)
    agg[key]["all"] += s
    tot["all"] += s
    for h in reasons:
        v = int(float(r[hdr.index(h)] or 0))
        agg[key][h] += v
        tot[h] += v
print("total samples", tot["all"], {k.replace("stall_", ""): v for k, v in tot.most_common(9) if k != "all"})
for key, c in sorted(agg.items(), key=lambda kv: -kv[1]["all"])[:top]:
    rs = ", ".join(f"{k.replace('stall_', '')}={v}" for k, v in c.most_common(5) if k != "all" and v)
    print(f"{c['all']:7d} {100.0 * c['all'] / tot['all']:5.1f}%  {key[0]}:{key[1]:<5d} {rs}")
