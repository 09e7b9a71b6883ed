"""Summarise gpurun_out ncu captures into committed profiles/.

usage: python scripts/make_profiles.py <tag> [round]
  reads gpurun_out/prof_<tag>.ncu-rep (ncu --set full) and gpurun_out/launches_<tag>.csv
  (ncu --metrics gpu__time_duration.sum launch list), writes
    profiles/r<round>_<tag>_ncu_full.json     per-kernel metrics of the full capture
    profiles/r<round>_<tag>_launches.md       launch list summary (time share per kernel)
    profiles/ncu_traffic.json                 {kernel: dram bytes per launch} read by bench.py
"""
import collections
import csv
import io
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "scripts"))
from ncu_summary import WANT  # noqa: E402


def short(name: str) -> str:
    m = re.search(r"(gat_[a-z_]+kernel|sgemm_kernel|gemm_tf32x3_kernel|[a-zA-Z_]+_kernel)(<[^>]*>)?", name)
    return (m.group(1) + (m.group(2) or "")) if m else name[:60]


def full_summary(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = {"kernel": short(r[hdr.index("Kernel Name")])}
        for w in WANT:
            if w in hdr:
                v = r[hdr.index(w)].replace(",", "")
                try:
                    d[w] = float(v)
                except ValueError:
                    d[w] = v
                d[w + ".unit"] = units[hdr.index(w)]
        out.append(d)
    return out


def launch_summary(path):
    txt = open(path).read()
    i = txt.find('"ID"')
    rows = list(csv.reader(io.StringIO(txt[i:])))
    hdr = rows[0]
    kn, mv, un = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for r in rows[1:]:
        if len(r) <= mv:
            continue
        v = float(r[mv].replace(",", ""))
        v = v / 1e6 if r[un] in ("ns", "nsecond") else (v / 1e3 if r[un] in ("us", "usecond") else v)  # -> ms
        k = short(r[kn])
        tot[k] += v
        cnt[k] += 1
    return tot, cnt


def main():
    tag = sys.argv[1]
    rnd = sys.argv[2] if len(sys.argv) > 2 else "01"
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    rep = os.path.join(ROOT, "gpurun_out", f"prof_{tag}.ncu-rep")
    traffic = {}
    if os.path.exists(rep):
        full = full_summary(rep)
        json.dump(full, open(os.path.join(ROOT, "profiles", f"r{rnd}_{tag}_ncu_full.json"), "w"), indent=1)
        name_map = {"gat_fwd_kernel": "gat_fwd", "gat_fwd_ovl_kernel": "gat_fwd", "gat_bwd_dst_kernel": "gat_bwd_dst",
                    "gat_bwd_src_kernel": "gat_bwd_src", "gat_bwd_src_fast_kernel": "gat_bwd_src_fused"}
        for d in full:
            base = d["kernel"].split("<")[0]
            if base in name_map and "dram__bytes_read.sum" in d:
                scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
                rd = d["dram__bytes_read.sum"] * scale.get(d["dram__bytes_read.sum.unit"], 1)
                wr = d["dram__bytes_write.sum"] * scale.get(d["dram__bytes_write.sum.unit"], 1)
                traffic.setdefault(name_map[base], rd + wr)
        if traffic:
            json.dump({**traffic, "_config": "bench.py default (reddit, fp32 gather, 1 GPU)",
                       "_source": f"profiles/r{rnd}_{tag}_ncu_full.json (ncu --set full, first launch)"},
                      open(os.path.join(ROOT, "profiles", "ncu_traffic.json"), "w"), indent=1)
    lpath = os.path.join(ROOT, "gpurun_out", f"launches_{tag}.csv")
    if os.path.exists(lpath):
        tot, cnt = launch_summary(lpath)
        allt = sum(tot.values())
        lines = [f"# launch list `{tag}` (ncu --metrics gpu__time_duration.sum --clock-control none; cold, serialised)",
                 "", "| kernel | launches | total ms | share |", "|---|---|---|---|"]
        for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
            lines.append(f"| `{k}` | {cnt[k]} | {v:.3f} | {100 * v / allt:.1f}% |")
        open(os.path.join(ROOT, "profiles", f"r{rnd}_{tag}_launches.md"), "w").write("\n".join(lines) + "\n")
    print("traffic:", traffic)


if __name__ == "__main__":
    main()
