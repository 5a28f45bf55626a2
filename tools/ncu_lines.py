"""Aggregate an ncu report's per-SASS stall samples / executed instructions
by CUDA source line, using the nvdisasm -g line table of the object file.
usage: python tools/ncu_lines.py REPORT.ncu-rep OBJECT.o KERNEL_SUBSTRING [N]"""
import collections, csv, io, os, re, subprocess, sys, tempfile

rep, obj, kname = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 25
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hi = [i for i, r in enumerate(rows) if r and r[0] == "Address"][0]
hdr = rows[hi]
data = [dict(zip(hdr, r)) for r in rows[hi + 1:] if len(r) == len(hdr)]
skey, ikey = "Warp Stall Sampling (All Samples)", "Instructions Executed"
with tempfile.TemporaryDirectory() as td:
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=td, capture_output=True)
    cub = [f for f in os.listdir(td) if f.endswith(".cubin")][0]
    dis = subprocess.run(["nvdisasm", "-g", os.path.join(td, cub)], capture_output=True, text=True).stdout
# walk the kernel's section: map instruction index -> line
lines = []
cur = None
inside = False
for ln in dis.splitlines():
    if ln.startswith("\t.section") or ln.startswith(".section"):
        inside = ".text." in ln and kname in ln
    if not inside:
        continue
    m = re.search(r"line (\d+)", ln)
    if m:
        cur = int(m.group(1))
    if re.search(r"/\*[0-9a-f]{4,}\*/", ln):
        lines.append(cur)
n = min(len(lines), len(data))
st, ins = collections.Counter(), collections.Counter()
for i in range(n):
    st[lines[i]] += float(data[i][skey] or 0)
    ins[lines[i]] += float(data[i][ikey] or 0)
ts, ti = sum(st.values()) or 1, sum(ins.values()) or 1
print(f"{len(lines)} disassembled vs {len(data)} profiled instructions")
for line, v in st.most_common(top):
    print(f"line {line}: stall {100 * v / ts:5.1f}%  inst {100 * ins[line] / ti:5.1f}%")
