"""Attribute shared-memory wavefronts (and the excess over ideal = bank conflicts) of one kernel
to CUDA source lines.  usage: python tools/smem_by_line.py REP.ncu-rep OBJ.o KERNEL_SUBSTR [top]"""
import collections, csv, io, os, re, subprocess, sys, tempfile

rep, obj, ksub = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr = rows[1]
ia, isrc = hdr.index("Address"), hdr.index("Source")
iw, ix, ie = hdr.index("L1 Wavefronts Shared"), hdr.index("L1 Wavefronts Shared Excessive"), hdr.index("Instructions Executed")
data = [r for r in rows[2:] if len(r) == len(hdr)]
base = int(data[0][ia], 16)
with tempfile.TemporaryDirectory() as td:
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=td, capture_output=True)
    lines = {}
    for cb in [f for f in os.listdir(td) if f.endswith(".cubin")]:
        dis = subprocess.run(["nvdisasm", "--print-line-info", "-c", os.path.join(td, cb)], capture_output=True, text=True).stdout
        fn = cur = None
        for ln in dis.splitlines():
            m = re.match(r"\s*\.text\.(\S+):", ln)
            if m:
                fn = m.group(1); continue
            m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
            if m:
                cur = (os.path.basename(m.group(1)), int(m.group(2))); continue
            m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
            if m and fn and ksub in fn:
                lines[int(m.group(1), 16)] = cur
num = lambda s: float(s.replace(",", "")) if s else 0.0
agg = collections.defaultdict(lambda: [0.0, 0.0, 0.0, collections.Counter()])
T = [0.0, 0.0]
for r in data:
    key = lines.get(int(r[ia], 16) - base, ("?", 0))
    w, x = num(r[iw]), num(r[ix])
    if w:
        a = agg[key]; a[0] += w; a[1] += x; a[2] += num(r[ie])
        a[3][r[isrc].split()[0] if r[isrc].split() else "?"] += 1
        T[0] += w; T[1] += x
print(f"total shared wavefronts {T[0]:.0f}, excessive {T[1]:.0f} ({100 * T[1] / max(T[0], 1):.1f} %)")
for key, a in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
    print(f"{key[0]}:{key[1]:<5d} wavefronts {a[0]:12.0f} excessive {a[1]:12.0f} ({100 * a[1] / max(a[0], 1):5.1f} %) inst {a[2]:10.0f} {dict(a[3])}")
