"""Sum ncu DRAM bytes / durations per hot-path operation (development
helper): pairs the kernels of an `ncu --page raw --csv` export of a
tools/kprof.py capture with the operation list kprof.py wrote (launch
order, launches per operation), and writes profiles/traffic_<cfg>.json.

    python tools/traffic_from_ncu.py c4 gpurun_out/kprof_c4_raw.csv gpurun_out/kprof_c4_ops.json
"""
import csv
import json
import sys


def main():
    key, raw, opsf = sys.argv[1:4]
    rows = list(csv.reader(open(raw)))
    # the first line that names the metric columns
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr, units, data = rows[h], rows[h + 1], rows[h + 2:]
    col = {name: hdr.index(name) for name in hdr}

    def val(r, name, scale_to=None):
        v = r[col[name]].replace(",", "")
        u = units[col[name]]
        x = float(v)
        if scale_to == "B":
            x *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(u, 1)
        if scale_to == "us":
            x *= {"nsecond": 1e-3, "usecond": 1, "msecond": 1e3, "second": 1e6}.get(u, 1)
        return x

    ops = json.load(open(opsf))
    kernels = []
    for r in data:
        if not r or len(r) < len(hdr):
            continue
        kernels.append({
            "name": r[col["Kernel Name"]].split("(")[0],
            "us": val(r, "gpu__time_duration.sum", "us"),
            "dram": val(r, "dram__bytes_read.sum", "B") + val(r, "dram__bytes_write.sum", "B"),
            "lts_pct": val(r, "lts__throughput.avg.pct_of_peak_sustained_elapsed"),
            "dram_pct": val(r, "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
            "warps_pct": val(r, "sm__warps_active.avg.pct_of_peak_sustained_active"),
            "regs": val(r, "launch__registers_per_thread"),
        })
    need = sum(o["launches"] for o in ops["ops"])
    if len(kernels) != need:
        print("warning: %d kernels captured, %d launches counted" % (len(kernels), need))
    out, i = {}, 0
    for o in ops["ops"]:
        ks = kernels[i:i + o["launches"]]
        i += o["launches"]
        us = sum(k["us"] for k in ks)
        dram = sum(k["dram"] for k in ks)
        out[o["op"]] = {
            "kernels": [k["name"] for k in ks],
            "ncu_us": round(us, 2),
            "dram_bytes": dram,
            "algorithmic_bytes": o["algorithmic_bytes"],
            "dram_over_algorithmic": round(dram / o["algorithmic_bytes"], 3),
            "dram_gbs_cold": round(dram / us / 1e3, 1) if us else None,
            "algorithmic_gbs_cold": round(o["algorithmic_bytes"] / us / 1e3, 1) if us else None,
            "per_kernel": [{k2: (round(v, 2) if isinstance(v, float) else v) for k2, v in k.items()} for k in ks],
        }
    doc = {
        "source": "ncu --set full --import-source on --clock-control none --profile-from-start off, "
                  "tools/kprof.py %s (each operation once, warm caches, between cudaProfilerStart/Stop); "
                  "ncu replays flush caches, so ncu_us is a cold-cache time" % key,
        "config": key, "m": ops["m"], "n": ops["n"], "nnz": ops["nnz"], "block": ops["block"],
        "dram_bytes_per_launch": {k: v["dram_bytes"] for k, v in out.items()},
        "ops": out,
    }
    json.dump(doc, open("profiles/traffic_%s.json" % key, "w"), indent=1)
    for k, v in out.items():
        print("%-24s %9.1f us  dram %8.3f GB  alg %8.3f GB  ratio %5.2f  %s" % (
            k, v["ncu_us"], v["dram_bytes"] / 1e9, v["algorithmic_bytes"] / 1e9, v["dram_over_algorithmic"],
            ",".join(sorted(set(v["kernels"])))[:90]))


if __name__ == "__main__":
    main()
