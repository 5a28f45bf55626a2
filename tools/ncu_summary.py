"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list:
per-kernel share of device time over the LAST `--steps` fraction of launches."""
import argparse, collections, csv

ap = argparse.ArgumentParser()
ap.add_argument("csv")
ap.add_argument("--tail-frac", type=float, default=0.5, help="fraction of launches (the timed step) to aggregate")
ap.add_argument("--top", type=int, default=25)
a = ap.parse_args()
rows = list(csv.reader(open(a.csv)))
hdr, data = None, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
sel = data[int(len(data) * (1 - a.tail_frac)):]
agg = collections.defaultdict(lambda: [0, 0.0])
for d in sel:
    name = d["Kernel Name"].split("(")[0].replace("unnamed>::", "")
    agg[name][0] += 1
    agg[name][1] += float(d["Metric Value"])
tot = sum(v[1] for v in agg.values())
unit = sel[0]["Metric Unit"] if sel else "?"
print(f"launches={len(sel)} total={tot/1e6 if unit=='ns' else tot:.3f} ms (serialised, cold-cache; compare shares)")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[: a.top]:
    ms = v[1] / 1e6 if unit == "ns" else v[1]
    print(f"{v[1]/tot*100:6.1f}%  {ms:9.3f} ms  n={v[0]:5d}  {k[:100]}")
