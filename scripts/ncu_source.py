"""Per-kernel SASS hot spots from an ncu report (source page): stall samples by opcode and top lines."""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
want = sys.argv[2] if len(sys.argv) > 2 else ""
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout.splitlines()
blocks, cur = [], None
for line in out:
    if line.startswith('"Kernel Name"'):
        cur = [line.split('","')[1].rstrip('",'), []]
        blocks.append(cur)
    elif cur is not None:
        cur[1].append(line)
for name, lines in blocks:
    if want not in name:
        continue
    rows = list(csv.reader(lines))
    hdr = rows[0]
    si, ii = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
    src = hdr.index("Source")
    stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    by_op = collections.Counter()
    by_op_stall = collections.defaultdict(collections.Counter)
    tot = 0
    for r in rows[1:]:
        if len(r) < len(hdr):
            continue
        op = r[src].split()[0] if r[src].split() else "?"
        if op.startswith("@"):
            op = r[src].split()[1]
        op = op.split(".")[0]
        s = int(r[si] or 0)
        by_op[op] += s
        tot += s
        for c in stall_cols:
            by_op_stall[op][hdr[c]] += int(r[c] or 0)
    print("=" * 20, name, "samples", tot, "instructions", len(rows) - 1)
    for op, s in by_op.most_common(14):
        top = ", ".join(f"{k[6:]}={v}" for k, v in by_op_stall[op].most_common(4))
        print(f"  {op:10s} {s:7d} {100 * s / max(tot, 1):5.1f}%  {top}")

if len(sys.argv) > 3:
    # dump the SASS with per-line samples for the first matching kernel
    for name, lines in blocks:
        if want not in name:
            continue
        rows = list(csv.reader(lines))
        hdr = rows[0]
        si, ii, src = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed"), hdr.index("Source")
        with open(sys.argv[3], "w") as f:
            for r in rows[1:]:
                if len(r) < len(hdr):
                    continue
                f.write(f"{r[si]:>6s} {r[ii]:>10s}  {r[src]}\n")
        break
