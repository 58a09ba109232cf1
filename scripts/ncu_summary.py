#!/usr/bin/env python
"""Summarise an ncu --set full report (one kernel launch) and an ncu launch list
into profiles/<round>/: key metrics, stall reasons, top source lines, launch
shares.  Usage: ncu_summary.py <report.ncu-rep> <launches.csv|-> <outdir> <config>"""
import csv, json, os, subprocess, sys
from collections import defaultdict

rep, lcsv, outdir, cfg = sys.argv[1:5]
os.makedirs(outdir, exist_ok=True)
raw = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h = rows[0]
KSEL = os.environ.get('NCU_KERNEL_ROW')  # which launch of a multi-kernel report (0-based)
v = rows[2 + int(KSEL)] if KSEL else rows[2]
m = dict(zip(h, v))
keys = ['Kernel Name', 'gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'dram__throughput.avg.pct_of_peak_sustained_elapsed', 'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread', 'launch__grid_size',
        'launch__block_size', 'launch__shared_mem_per_block_dynamic', 'lts__t_sector_hit_rate.pct', 'smsp__inst_executed.sum',
        'smsp__sass_thread_inst_executed_op_dfma_pred_on.sum', 'smsp__sass_thread_inst_executed_op_dadd_pred_on.sum',
        'smsp__sass_thread_inst_executed_op_dmul_pred_on.sum']
units = dict(zip(h, rows[1]))
summ = {k: (m.get(k), units.get(k)) for k in keys if k in m}
stalls = {k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', ''): float(x)
          for k, x in m.items() if k.startswith('smsp__average_warps_issue_stalled_') and k.endswith('ratio')
          and x and float(x) > 0.02}
def num(k):
    x, u = summ[k]
    f = float(x.replace(',', ''))
    return f * {'Gbyte': 1e9, 'Mbyte': 1e6, 'Kbyte': 1e3, 'byte': 1, 'Tbyte': 1e12}.get(u, 1)
traffic = num('dram__bytes_read.sum') + num('dram__bytes_write.sum')
# source lines
cs = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'cuda,sass'], capture_output=True,
                    text=True).stdout
agg = {}
f = None
for r in csv.reader(cs.splitlines()):
    if r and r[0] == 'File Path': f = r[1].split('/')[-1]; continue
    if not r or r[0] == 'Line No' or len(r) < 8: continue
    try: s_, e_ = float(r[4] or 0), float(r[7] or 0)
    except ValueError: continue
    a = agg.setdefault((f, r[0]), [0, 0, r[1][:90]]); a[0] += s_; a[1] += e_
    if r[1].strip(): a[2] = r[1][:90]
tot = sum(x[0] for x in agg.values()) or 1; totE = sum(x[1] for x in agg.values()) or 1
lines = [f"{x[0]/tot*100:5.1f}% stall {x[1]/totE*100:5.1f}% inst  {k[0]}:{k[1]}  {x[2]}"
         for k, x in sorted(agg.items(), key=lambda kv: -kv[1][0])[:30]]
launches = []
if lcsv != '-' and os.path.exists(lcsv):
    hd = None; acc = defaultdict(lambda: [0, 0.0])
    for r in csv.reader(open(lcsv)):
        if r and r[0] == 'ID': hd = r; continue
        if hd and len(r) == len(hd):
            d = dict(zip(hd, r))
            if d['Metric Name'] == 'gpu__time_duration.sum':
                a = acc[d['Kernel Name']]; a[0] += 1; a[1] += float(d['Metric Value'].replace(',', ''))
    t = sum(x[1] for x in acc.values()) or 1
    launches = [f"{x[0]:5d} launches {x[1]/1e3:11.1f} us total {x[1]/max(1,x[0])/1e3:10.1f} us/launch {x[1]/t*100:5.1f}%  {k[:100]}"
                for k, x in sorted(acc.items(), key=lambda kv: -kv[1][1])]
kshort = m['Kernel Name'].split('(')[0].split('::')[-1].split('<')[0]
suffix = f"_{kshort}" if KSEL else ""
with open(os.path.join(outdir, f'ncu_{cfg}{suffix}_summary.txt'), 'w') as o:
    o.write(f"ncu --set full --clock-control none, one launch ({rep})\n\n")
    for k, (x, u) in summ.items(): o.write(f"{k:70s} {x} {u or ''}\n")
    o.write(f"\nDRAM traffic per launch (read + write): {traffic/1e9:.3f} GB\n\nstall reasons (warps per issue):\n")
    for k, x in sorted(stalls.items(), key=lambda kv: -kv[1]): o.write(f"  {k:30s} {x:.3f}\n")
    o.write("\ntop source lines by stall samples:\n" + "\n".join(lines) + "\n")
    if launches:
        o.write(f"\nlaunch list ({lcsv}; ncu --metrics gpu__time_duration.sum, cold-cache, serialised; whole process incl. one-time symbolic phase):\n")
        o.write("\n".join(launches) + "\n")
tp = os.path.join(os.path.dirname(outdir.rstrip('/')), 'ncu_traffic.json')
tj = json.load(open(tp)) if os.path.exists(tp) else {}
kn = kshort
tj[f"{cfg}:{kn}"] = traffic
json.dump(tj, open(tp, 'w'), indent=1, sort_keys=True)
print(open(os.path.join(outdir, f'ncu_{cfg}{suffix}_summary.txt')).read()[:1500])
