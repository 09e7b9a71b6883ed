"""Aggregate an ncu source page (SASS) by opcode: stall samples and executed instructions.
usage: sass_hotspots.py report.ncu-rep kernel_regex [launch_skip]"""
import collections, csv, io, subprocess, sys

rep, kre = sys.argv[1], sys.argv[2]
skip = sys.argv[3] if len(sys.argv) > 3 else "0"
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kre}",
                      "--launch-skip", skip, "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
i0 = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
hdr = rows[i0]
iS, iI, iSrc = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed"), hdr.index("Source")
st, ins = collections.Counter(), collections.Counter()
seq = []
for r in rows[i0 + 1:]:
    if len(r) <= iI:
        continue
    op = r[iSrc].split()[0] if r[iSrc].split() else "?"
    if op.startswith("@"):
        op = r[iSrc].split()[1]
    op = op.split(".")[0]
    try:
        s, n = float(r[iS] or 0), float(r[iI] or 0)
    except ValueError:
        continue
    st[op] += s
    ins[op] += n
    seq.append((s, r[iSrc][:80]))
ts, ti = sum(st.values()), sum(ins.values())
print(f"total stall samples {ts:.0f}, instructions {ti:.3e}")
for op, s in st.most_common(18):
    print(f"{op:10s} stall {100 * s / ts:5.1f}%  inst {100 * ins[op] / ti:5.1f}%")
print("top instructions by stall:")
for s, src in sorted(seq, reverse=True)[:15]:
    print(f"  {100 * s / ts:5.1f}%  {src}")
