"""Summarise the ncu captures of a round into profiles/ncu_summary.json.

Inputs (written by the round's gpurun profile call, scratch paths):
  --rep     an `ncu --set full` report of one bench layer (qkv launch, o launch)
  --launch  the `--metrics gpu__time_duration.sum` launch-list CSV of a short
            bench run (every kernel of the timed steps, cold and serialised)
Output: the per-launch DRAM traffic that bench.py reports as roofline.traffic,
the key SOL metrics of the captured launches and the launch-list shares.
"""
import argparse
import csv
import io
import json
import subprocess
import sys

WANT = {
    "gpu__time_duration.sum": "duration_ns",
    "dram__bytes_read.sum": "dram_read_bytes",
    "dram__bytes_write.sum": "dram_write_bytes",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "sm__inst_executed.sum": "warp_instructions",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "lts__t_bytes.sum": "l2_bytes",
}
UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3, "msecond": 1e6,
              "ns": 1, "us": 1e3}


def raw_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, body = rows[0], rows[1], rows[2:]
    kernels = []
    for r in body:
        k = {"name": r[hdr.index("Kernel Name")]}
        for m, key in WANT.items():
            if m in hdr:
                i = hdr.index(m)
                try:
                    v = float(r[i].replace(",", ""))
                except ValueError:
                    continue
                k[key] = v * UNIT_SCALE.get(units[i], 1)
        kernels.append(k)
    return kernels


def launch_list(path):
    durs = {}
    txt = open(path).read().splitlines()
    start = next(i for i, l in enumerate(txt) if l.startswith('"ID"'))
    for r in csv.DictReader(txt[start:]):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"]
        v = float(r["Metric Value"].replace(",", "")) * UNIT_SCALE.get(r.get("Metric Unit", "ns"), 1)
        durs.setdefault(name, []).append(v)
    tot = sum(sum(v) for v in durs.values())
    return {n: {"launches": len(v), "total_us": round(sum(v) / 1e3, 2), "mean_us": round(sum(v) / len(v) / 1e3, 2),
                "share": round(sum(v) / tot, 4)} for n, v in sorted(durs.items(), key=lambda kv: -sum(kv[1]))}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep", required=True)
    ap.add_argument("--launch", default=None)
    ap.add_argument("--workload", required=True)
    ap.add_argument("--alg-bytes", default=None, help="json {qkv: B, o: B} algorithmic bytes per launch")
    ap.add_argument("--round", default="r01")
    ap.add_argument("--out", default="profiles/ncu_summary.json")
    a = ap.parse_args()
    ks = raw_metrics(a.rep)
    labels = ["qkv", "o"]
    per = {}
    for lab, k in zip(labels, ks):
        k["dram_bytes"] = k.get("dram_read_bytes", 0) + k.get("dram_write_bytes", 0)
        per[lab] = k
    summ = {"round": a.round, "workload": a.workload,
            "source": "ncu --set full --clock-control none (one layer: qkv launch, o launch; cold, serialised)",
            "dram_bytes_per_launch": {lab: per[lab]["dram_bytes"] for lab in per},
            "launches": per}
    if a.alg_bytes:
        alg = json.loads(a.alg_bytes)
        summ["alg_bytes_per_launch"] = alg
        summ["dram_over_alg"] = {lab: round(per[lab]["dram_bytes"] / alg[lab], 3) for lab in per if lab in alg}
    if a.launch:
        summ["launch_list"] = launch_list(a.launch)
    json.dump(summ, open(a.out, "w"), indent=1)
    json.dump(summ, sys.stdout, indent=1)


if __name__ == "__main__":
    main()
