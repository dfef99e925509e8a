"""Summarise `ncu --page raw --csv` exports (one per kernel) into profiles/traffic.json and a markdown table.

usage: python tools/ncu_summarise.py <dir with *_raw.csv> <traffic.json> <summary.md>
"""
import csv
import glob
import json
import os
import sys

UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
        "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0, "second": 1.0}


def load(path):
    rows = list(csv.reader(open(path)))
    if len(rows) < 3:
        return None
    head, units, vals = rows[0], rows[1], rows[2]
    out = {}
    for h, u, v in zip(head, units, vals):
        out[h] = (v, u)
    return out


def num(m, key, default=None):
    if key not in m:
        return default
    v, u = m[key]
    try:
        x = float(v.replace(",", ""))
    except ValueError:
        return default
    return x * UNIT.get(u, 1.0)


def first(m, keys, default=None):
    for k in keys:
        x = num(m, k)
        if x is not None:
            return x
    return default


def main(src, out_json, out_md):
    res = {}
    for p in sorted(glob.glob(os.path.join(src, "*_raw.csv"))):
        k = os.path.basename(p)[:-len("_raw.csv")]
        m = load(p)
        if m is None:
            continue
        rd, wr = num(m, "dram__bytes_read.sum", 0.0), num(m, "dram__bytes_write.sum", 0.0)
        res[k] = {
            "dram_bytes": rd + wr, "dram_read": rd, "dram_write": wr,
            "ncu_duration_s": num(m, "gpu__time_duration.sum"),
            "fp64_pipe_pct": first(m, ["sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
                                       "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"]),
            "warps_active_pct": num(m, "sm__warps_active.avg.pct_of_peak_sustained_active"),
            "l2_hit_pct": num(m, "lts__t_sector_hit_rate.pct"),
            "registers": num(m, "launch__registers_per_thread"),
            "smem_bank_conflicts": first(m, ["l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]),
            "smem_wavefronts": first(m, ["l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"]),
            "local_load_sectors": first(m, ["l1tex__t_sectors_pipe_lsu_mem_local_op_ld.sum"]),
            "local_store_sectors": first(m, ["l1tex__t_sectors_pipe_lsu_mem_local_op_st.sum"]),
        }
    json.dump(res, open(out_json, "w"), indent=1)
    with open(out_md, "w") as f:
        f.write("| kernel | duration ms | DRAM GB | DRAM GB/s | FP64 pipe % | warps active % | L2 hit % | regs | "
                "smem bank conflicts / wavefronts | local ld/st sectors |\n|---|---|---|---|---|---|---|---|---|---|\n")
        for k, r in sorted(res.items(), key=lambda kv: -(kv[1]["ncu_duration_s"] or 0)):
            d = r["ncu_duration_s"] or float("nan")
            fmt = lambda x, s="%.1f": "-" if x is None else s % x
            f.write(f"| {k} | {d*1e3:.3f} | {r['dram_bytes']/1e9:.3f} | {r['dram_bytes']/1e9/d:.0f} | "
                    f"{fmt(r['fp64_pipe_pct'])} | {fmt(r['warps_active_pct'])} | {fmt(r['l2_hit_pct'])} | "
                    f"{fmt(r['registers'], '%d')} | {fmt(r['smem_bank_conflicts'], '%d')} / {fmt(r['smem_wavefronts'], '%d')} | "
                    f"{fmt(r['local_load_sectors'], '%d')} / {fmt(r['local_store_sectors'], '%d')} |\n")
    print(open(out_md).read())


if __name__ == "__main__":
    main(*sys.argv[1:4])
