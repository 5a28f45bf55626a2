"""Extract the roofline metrics of one launch from an ncu --set full report
(via `ncu -i REP --page raw --csv`) into a committed JSON summary.
Usage: ncu_to_json.py REP INDEX OUT.json "kernel label" "command" ALG_BYTES [ALG_FLOPS]"""
import csv, io, json, subprocess, sys

rep, idx, out, label, cmd, alg_bytes = sys.argv[1], int(sys.argv[2]), sys.argv[3], sys.argv[4], sys.argv[5], float(sys.argv[6])
alg_flops = float(sys.argv[7]) if len(sys.argv) > 7 else None
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, data = rows[0], rows[1], rows[2:]
r = data[idx]
keep = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__cycles_elapsed.avg.per_second", "launch__grid_size", "launch__registers_per_thread",
        "launch__shared_mem_per_block_dynamic"]
m = {}
for k in keep:
    if k in hdr:
        i = hdr.index(k)
        m[k] = {"value": r[i], "unit": units[i]}
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
def b(k):
    return float(m[k]["value"].replace(",", "")) * scale[m[k]["unit"]]
res = {"kernel": label, "command": cmd, "dram_bytes_per_launch": b("dram__bytes_read.sum") + b("dram__bytes_write.sum"),
       "dram_read_bytes": b("dram__bytes_read.sum"), "dram_write_bytes": b("dram__bytes_write.sum"),
       "algorithmic_bytes_per_launch": alg_bytes, "metrics": m}
if alg_flops:
    res["algorithmic_flops_per_launch"] = alg_flops
json.dump(res, open(out, "w"), indent=1)
print(json.dumps({k: v for k, v in res.items() if k != "metrics"}, indent=1))
print({k: v["value"] for k, v in m.items()})
