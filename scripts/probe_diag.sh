mkdir -p gpurun_out; python scripts/probe_diag.py ${CFG:-deep} 16 > gpurun_out/diag.log 2>&1; tail -8 gpurun_out/diag.log; ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_probe --csv --log-file gpurun_out/diag_launch.csv python scripts/probe_diag.py ${CFG:-deep} 16 > gpurun_out/diag_ncu.log 2>&1; python3 -c "
import csv
r=list(csv.reader(open('gpurun_out/diag_launch.csv')))
h=None
for row in r:
    if 'Kernel Name' in row: h=row; continue
    if h and len(row)==len(h): print(row[h.index('Kernel Name')][:20], row[-1])
" | tail -6
