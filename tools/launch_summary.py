"""Per-kernel totals of an ncu launch list (--metrics gpu__time_duration.sum --csv), per pass.

Stage 1 runs in batches of up to 8 passes that are enqueued ahead of Stage 2 (a profiled run of
P Stage-2 passes holds the Stage-1 work of more than P passes: the ramp 1, 2, 4, 8 plus the
look-ahead batch), so each stage is normalised by ITS OWN pass count: Stage-2 kernels by the
number of k_conn_mis launches, Stage-1 kernels by the passes of the batches in the list
(k_pool_select's grid = passes of the batch). A Stage-1 batch is a contiguous run of launches
in the list: pool-walk wavefront (k_light_start, traversal + k_shade* per bounce), k_pool_keys,
selection, entries, probes, bounds, the reciprocal rounds, k_pool_finish.

  python tools/launch_summary.py launches.csv [top]
"""
import collections
import csv
import sys


def short(name):
    return name.split("(")[0].replace("void ", "").split("::")[-1][:48]


def main():
    rows = [r for r in csv.DictReader(l for l in open(sys.argv[1]) if l.startswith('"'))
            if r["Metric Name"] == "gpu__time_duration.sum"]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}
    names = [short(r["Kernel Name"]) for r in rows]
    ms = [float(r["Metric Value"].replace(",", "")) * scale[r["Metric Unit"]] for r in rows]
    stage1 = [False] * len(rows)
    s1_passes = 0
    for i, n in enumerate(names):
        if n != "k_pool_keys":
            continue
        a = i
        while a > 0 and (names[a - 1].startswith("k_trav_persistent") or names[a - 1].startswith("k_shade")):
            a -= 1
        if a > 0 and names[a - 1] == "k_light_start":
            a -= 1
        b = i
        seen_finish = False
        while b + 1 < len(names):
            nxt = names[b + 1]
            if seen_finish and nxt != "k_pool_finish":
                break
            seen_finish = seen_finish or nxt == "k_pool_finish"
            b += 1
        for k in range(a, b + 1):
            stage1[k] = True
            if names[k] == "k_pool_select":
                grid = rows[k]["Grid Size"].strip("()").split(",")[0]
                s1_passes += int(grid)
    s2_passes = names.count("k_conn_mis") or 1
    s1_passes = s1_passes or 1
    agg = collections.defaultdict(lambda: [0, 0.0])
    for n, t, s1 in zip(names, ms, stage1):
        key = ("S1 " if s1 else "S2 ") + n
        agg[key][0] += 1
        agg[key][1] += t / (s1_passes if s1 else s2_passes)
    t1 = sum(v[1] for k, v in agg.items() if k.startswith("S1"))
    t2 = sum(v[1] for k, v in agg.items() if k.startswith("S2"))
    tot = t1 + t2
    print(f"{len(rows)} launches: {s2_passes} Stage-2 passes, {s1_passes} Stage-1 passes (batched ahead)")
    print(f"serialised per pass: Stage 2 {t2:.3f} ms + Stage 1 {t1:.3f} ms = {tot:.3f} ms")
    recip = sum(v[1] for k, v in agg.items() if k.startswith("S1") and
                ("k_rq_" in k or "k_recip_" in k or
                 ("k_trav_persistent" in k and False)))
    # the reciprocal rounds' traversal launches: Stage-1 traversal after k_recip_init
    rt = 0.0
    in_recip = False
    for n, t, s1 in zip(names, ms, stage1):
        if not s1:
            in_recip = False
            continue
        if n == "k_recip_init":
            in_recip = True
        elif n == "k_pool_finish":
            in_recip = False
        if in_recip and n.startswith("k_trav_persistent"):
            rt += t / s1_passes
    print(f"reciprocal estimation (node evaluation + its traversal + DFS): {recip + rt:.3f} ms per pass "
          f"= {100 * (recip + rt) / tot:.1f}% (traversal part {rt:.3f} ms)")
    for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        print(f"{v:8.3f} ms/pass {100 * v / tot:5.1f}% {c:6d} {k}")


if __name__ == "__main__":
    main()
