"""Summarise the Gram-Schmidt kernels of one 4096^2 FGMRES solve from an ncu
launch list (tools/krylov_ncu.sh): per launch the time, DRAM bytes, the number
of vectors streamed (algorithmic: k_cgs_dots reads its mm vectors, k_cgs_update
reads m basis vectors + w and writes w_out), achieved algorithmic GB/s and the
DRAM/algorithmic ratio.

    python tools/krylov_summary.py gpurun_out/krylov_launches_r2b.csv [N] [hbm_peak_gbs]
"""
import csv
import json
import sys
from collections import OrderedDict


def main():
    path = sys.argv[1]
    N = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
    peak = float(sys.argv[3]) if len(sys.argv) > 3 else 6538.3
    lat = 2 * N + 1
    pu = (lat + 7) // 8 * 8
    pp = (N + 1 + 7) // 8 * 8
    n_el = 2 * lat * pu + (N + 1) * pp  # elements a pass streams (owned rows incl. pitch padding)
    vec = 8.0 * n_el
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    I = {k: hdr.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Value", "Metric Unit")}
    L = OrderedDict()
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "ns": 1e-9, "usecond": 1e-6, "us": 1e-6, "msecond": 1e-3, "ms": 1e-3,
             "second": 1.0}
    for r in rows[h + 1:]:
        if len(r) < len(hdr):
            continue
        d = L.setdefault(r[I["ID"]], {"kernel": r[I["Kernel Name"]].split("(")[0]})
        v = float(r[I["Metric Value"]].replace(",", "")) * scale.get(r[I["Metric Unit"]], 1.0)
        d[r[I["Metric Name"]]] = v
    out = []
    agg = {}
    for k, d in L.items():
        t = d["gpu__time_duration.sum"]
        rd, wr = d.get("dram__bytes_read.sum", 0.0), d.get("dram__bytes_write.sum", 0.0)
        upd = "update" in d["kernel"]
        nread = max(1, round(rd / vec))            # vectors the launch streamed from DRAM
        alg = (nread + (1 if upd else 0)) * vec    # + w_out written by an update
        rec = {"id": k, "kernel": d["kernel"], "ms": 1e3 * t, "vectors_read": nread, "alg_bytes": alg,
               "dram_bytes": rd + wr, "dram_over_alg": (rd + wr) / alg, "alg_gbs": alg / t / 1e9,
               "frac_of_measured_hbm": alg / t / 1e9 / peak}
        out.append(rec)
        a = agg.setdefault(d["kernel"], {"launches": 0, "ms": 0.0, "alg_bytes": 0.0, "dram_bytes": 0.0})
        a["launches"] += 1
        a["ms"] += 1e3 * t
        a["alg_bytes"] += alg
        a["dram_bytes"] += rd + wr
    for a in agg.values():
        a["alg_gbs"] = a["alg_bytes"] / (a["ms"] * 1e-3) / 1e9
        a["frac_of_measured_hbm"] = a["alg_gbs"] / peak
        a["dram_over_alg"] = a["dram_bytes"] / a["alg_bytes"]
    print(json.dumps({"N": N, "vector_bytes": vec, "hbm_peak_gbs": peak,
                      "note": "cold-cache serialised ncu replays (--clock-control none); algorithmic bytes = "
                              "vectors streamed x vector bytes",
                      "per_kernel": agg, "launches": out}, indent=1))


if __name__ == "__main__":
    main()
