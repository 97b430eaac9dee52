"""Summarise an ncu --set full report: key metrics and stall reasons per kernel.

    python tools/ncu_summary.py gpurun_out/prof_x.ncu-rep [--json out.json --key c4]
"""
import csv
import io
import json
import subprocess
import sys

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "launch__registers_per_thread", "launch__block_size", "launch__grid_size",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "sm__cycles_active.avg",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
        "smsp__inst_executed_op_shared_atom.sum"]


def main():
    rep = sys.argv[1]
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = {}
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")]
        short = "gather" if "k_gather" in name else ("scatter" if "k_scatter" in name else name[:40])
        d = {}
        for w in WANT:
            if w in hdr:
                v = r[hdr.index(w)].replace(",", "")
                try:
                    d[w] = float(v)
                except ValueError:
                    d[w] = v
                d[w + "_unit"] = units[hdr.index(w)]
        stalls = {}
        for i, h in enumerate(hdr):
            if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
                try:
                    v = float(r[i].replace(",", ""))
                except ValueError:
                    continue
                if v > 0.05:
                    stalls[h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = v
        d["stalls_per_issue"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1]))
        res[short] = d
        print(f"== {short}: {name[:90]}")
        for k, v in d.items():
            if not k.endswith("_unit"):
                print(f"   {k} = {v} {d.get(k + '_unit', '')}")
    if "--json" in sys.argv:
        path = sys.argv[sys.argv.index("--json") + 1]
        key = sys.argv[sys.argv.index("--key") + 1]
        try:
            allj = json.load(open(path))
        except Exception:
            allj = {}
        allj.setdefault(key, {})
        byte_scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
        time_scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0,
                      "second": 1e3, "s": 1e3}
        for k, d in res.items():
            gb = sum(d.get(mn, 0) * byte_scale.get(d.get(mn + "_unit"), 1.0)
                     for mn in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
            tm = d.get("gpu__time_duration.sum")
            tm = tm * time_scale.get(d.get("gpu__time_duration.sum_unit"), 1.0) if tm is not None else None
            allj[key]["gather_apply" if k == "gather" else k] = {
                "dram_bytes_per_launch": gb, "report": rep,
                "time_ms": tm,
                "smem_wavefronts_per_launch": d.get("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"),
                "smem_pipe_pct_of_peak": d.get("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"),
                "smem_atom_wavefronts": d.get("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum"),
                "smem_atom_bank_conflicts": d.get("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom.sum"),
                "smem_atom_instructions": d.get("smsp__inst_executed_op_shared_atom.sum"),
                "sm_cycles_active": d.get("sm__cycles_active.avg")}
        json.dump(allj, open(path, "w"), indent=1)


if __name__ == "__main__":
    main()
