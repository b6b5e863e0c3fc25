"""Prints the numbers quoted in profiles/r2/r2_ncu_summary.md and DESIGN.md §8a from an evidence
directory written by tools/jobs/final.sh (bench_*.json, launch_shares_*.txt, C4_*_raw.csv)."""
import csv
import json
import os
import sys

d = sys.argv[1]
for cfg in ("C1", "C3", "C4", "C5"):
    p = os.path.join(d, f"bench_{cfg}.json")
    if not os.path.exists(p):
        continue
    x = json.load(open(p))
    r = x["roofline"]
    print(cfg, "value", round(x["value"], 2), "ms", round(x["ms_per_step"], 2), "e2e",
          x["e2e"]["value"] if x.get("e2e") else None, "spp", x["e2e"]["spp"] if x.get("e2e") else None, "hbm_frac",
          r["frac"], "l2_frac", r["l2"]["frac"], "bytes/ray", r["per_kernel"]["closest"]["bytes_per_ray"], "hbm_gb",
          x["hbm_gb_used"], "eval/cons", x["recip_nodes"]["evaluated_per_consumed"])
    if cfg == "C4":
        c2 = x["C2"]
        print("C2", "value", round(c2["value"], 2), "ms", round(c2["ms_per_step"], 3), "hbm_frac", c2["roofline"]["frac"],
              "l2_frac", c2["roofline"]["l2"]["frac"], "hbm_gb", c2["hbm_gb_used"])
        print("cpu_baseline", x["cpu_baseline"]["value"], "launches", x["gpu_launches"], "clocks", x["clocks"])
p = os.path.join(d, "bench_reference_C4.json")
if os.path.exists(p):
    print("reference arm", json.load(open(p))["value"])
for cfg in ("C4", "C2"):
    p = os.path.join(d, f"launch_shares_{cfg}.txt")
    if os.path.exists(p):
        print("".join(open(p).readlines()[:16]))
for k in ("trav0", "shade", "rq_setup", "rq_record", "rq_glue", "dfs"):
    p = os.path.join(d, f"C4_{k}_raw.csv")
    if not os.path.exists(p):
        continue
    rows = list(csv.reader(open(p)))
    m = dict(zip(rows[0], rows[2]))
    u = dict(zip(rows[0], rows[1]))
    g = lambda n: m.get(n, "?")
    print(k, "dur", g("gpu__time_duration.sum"), u.get("gpu__time_duration.sum"), "regs", g("launch__registers_per_thread"),
          "lanes", g("smsp__thread_inst_executed_per_inst_executed.ratio"), "occ",
          g("sm__warps_active.avg.pct_of_peak_sustained_active"), "issue", g("smsp__issue_active.avg.per_cycle_active"),
          "l1", g("l1tex__t_sector_hit_rate.pct"), "l2", g("lts__t_sector_hit_rate.pct"), "dramR",
          g("dram__bytes_read.sum"), u.get("dram__bytes_read.sum"), "dramW", g("dram__bytes_write.sum"),
          u.get("dram__bytes_write.sum"), "inst", g("smsp__inst_executed.sum"))
