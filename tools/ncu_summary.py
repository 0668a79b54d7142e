"""Summarise ncu --set full raw CSV exports (DRAM bytes, duration, DMMA pipe)
and refresh profiles/r02_traffic.json entries.
  python tools/ncu_summary.py gpurun_out/ncu_cb sinv:c2_pobtasi pobtaf_c2:c2_pobtaf \
      pobtaf_c3:c3shape_pobtaf_n12_b5026_a3"""
import csv
import json
import os
import sys

KEYS = {"dram__bytes_read.sum": "read", "dram__bytes_write.sum": "write",
        "gpu__time_duration.sum": "time",
        "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active": "dmma"}
SCALE = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "ms": 1.0, "us": 1e-3, "%": 1.0}


def read(path):
    rows = list(csv.reader(open(path)))
    hdr, units, vals = rows[0], rows[1], rows[-1]
    out = {}
    for h, u, v in zip(hdr, units, vals):
        if h in KEYS:
            out[KEYS[h]] = float(v.replace(",", "")) * SCALE.get(u, 1.0)
    return out


def main():
    d = sys.argv[1]
    tpath = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                         "profiles", "r02_traffic.json")
    table = json.load(open(tpath))
    for spec in sys.argv[2:]:
        name, key = spec.split(":")
        m = read(os.path.join(d, f"{name}_raw.csv"))
        print(f"{name}: {m['time']:.2f} ms, DRAM {m['read']/1e9:.2f} + {m['write']/1e9:.2f} GB, "
              f"DMMA pipe {m['dmma']:.1f}%")
        ent = table.setdefault(key, {})
        ent.update({"dram_bytes": int(m["read"] + m["write"]), "ms": round(m["time"], 2),
                    "dmma_pipe_pct": round(m["dmma"], 2)})
    json.dump(table, open(tpath, "w"), indent=1)


if __name__ == "__main__":
    main()
