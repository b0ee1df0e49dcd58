"""Per-group instruction accounting of the row-table kernel's hot loop from an ncu --set full
report's SASS source page (executed-instruction counts): the loop body is the contiguous region
whose instructions execute once per 4-node group; the spin-wait on the row pipeline executes
more often.  Usage: sass_hotloop.py report.ncu-rep > summary.txt"""
import collections, csv, io, subprocess, sys
raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, data = rows[1], rows[2:]
isrc, iex, iss = hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
ex = [int(r[iex]) for r in data]
mx = max(ex)
def op(s):
    t = s.strip().split()
    return (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
spin = max(range(len(data)), key=lambda i: ex[i])           # the spin loop runs most often
# the group body: instructions executing at the per-group rate (the most common count)
cnt = collections.Counter(e for e in ex if e > 0.02 * mx)
per_group = max(cnt, key=lambda e: cnt[e] * e if e < 0.5 * mx else 0)
groups = sum(1 for e in ex if abs(e - per_group) <= 0.02 * per_group)
tot = sum(ex)
c = collections.Counter()
for r in data:
    c[op(r[isrc])] += int(r[iex])
print(f"# SASS hot-loop accounting of {sys.argv[1]}")
print(f"instructions executed: {tot}; per-group execution count ~{per_group} (x2 orientations)")
print(f"warp-instructions per 4-node group (all regions / group executions): {tot / (2 * per_group):.1f}")
print("by opcode, per group:", ", ".join(f"{k} {v / (2 * per_group):.1f}" for k, v in c.most_common(18)))
print(f"spin loop: {ex[spin] / per_group:.1f} iterations per group ({op(data[spin][isrc])} at the most-executed address)")
