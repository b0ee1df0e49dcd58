#!/bin/bash
# r2p: ncu --set full of the lean general-stencil queue kernel on the C3 STATIC solve (every CTA busy)
timeout 1800 ncu --set full --import-source on --clock-control none -k regex:k_sweep_queue --launch-skip 0 --launch-count 1 \
    -o /tmp/prof_r2p_c3s -f python scripts/explore.py --cfg C3 --tol 1e-7 --schedule queue --modes static > gpurun_out/r2p_ncu.log 2>&1
python scripts/ncu_summary.py /tmp/prof_r2p_c3s.ncu-rep gpurun_out/r2p_sweep_queue_C3_static_ncu_summary.txt > /dev/null 2>&1
ncu -i /tmp/prof_r2p_c3s.ncu-rep --page source --csv > /tmp/src.csv 2>/dev/null
python - <<'PY'
import csv, collections
rows = list(csv.reader(open('/tmp/src.csv')))
hdr = rows[0]
print(hdr[:12])
# find columns
def col(name):
    for i, h in enumerate(hdr):
        if h.strip() == name: return i
    return None
ci = {k: col(k) for k in ("Source", "# Instructions Executed" , "Instructions Executed", "Warp Stall Sampling (All Samples)", "Address")}
print(ci)
si = ci["Warp Stall Sampling (All Samples)"]; ii = ci["Instructions Executed"] or ci["# Instructions Executed"]; so = ci["Source"]
data = []
for r in rows[1:]:
    try: data.append((int(r[si] or 0), int(r[ii] or 0), r[so]))
    except Exception: pass
tot_s = sum(d[0] for d in data) or 1; tot_i = sum(d[1] for d in data) or 1
out = open('gpurun_out/r2p_c3_static_hot_sass.txt', 'w')
out.write(f"total stall samples {tot_s}, instructions {tot_i}\n")
for s_, i_, src in sorted(data, key=lambda x: -x[0])[:60]:
    out.write(f"{100*s_/tot_s:6.2f}% samples {100*i_/tot_i:6.2f}% inst  {src}\n")
opc = collections.Counter()
for s_, i_, src in data:
    op = src.split()[0] if src.split() else '?'
    if op.startswith('@'): op = src.split()[1]
    opc[op.split('.')[0]] += i_
out.write("\ninstruction mix (executed):\n")
for k, v in opc.most_common(25): out.write(f"{100*v/tot_i:6.2f}%  {k}\n")
PY
