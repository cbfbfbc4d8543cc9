"""Per-launch time, occupancy, issue, FP64 pipe, DRAM bytes, active lanes and the top warp
stall reasons from `ncu --page raw --csv` exports (launches >= 50 us):
    python tools/ncu_stall_summary.py raw1.csv [raw2.csv ...]"""
import csv, sys
def f(v):
    try: return float(v.replace(',',''))
    except: return None
for fn in sys.argv[1:]:
    rows=list(csv.reader(open(fn)))
    hdr=rows[0]; units=rows[1]
    ki=hdr.index('Kernel Name'); ti=hdr.index('gpu__time_duration.sum')
    tu=units[ti]
    print('==', fn, tu)
    for r in rows[2:]:
        t=f(r[ti]); 
        if t is None: continue
        if tu=='us': t/=1000
        if t<0.05: continue
        d=dict(zip(hdr,r))
        def g(k):
            return f(d.get(k,'')) or 0
        dr=g('dram__bytes_read.sum'); dw=g('dram__bytes_write.sum')
        ur=units[hdr.index('dram__bytes_read.sum')]
        sc={'byte':1,'Kbyte':1e3,'Mbyte':1e6,'Gbyte':1e9}.get(ur,1)
        st=[(f(v),k.replace('smsp__average_warps_issue_stalled_','').replace('_per_issue_active.ratio','')) for k,v in d.items() if k.startswith('smsp__average_warps_issue_stalled') and f(v)]
        st=sorted(st,reverse=True)[:3]
        print(f"{r[ki][:34]:34s} {t:7.3f}ms regs={d.get('launch__registers_per_thread')} occ={g('sm__warps_active.avg.pct_of_peak_sustained_active'):.0f}% issue={g('smsp__issue_active.avg.pct_of_peak_sustained_active'):.0f}% fp64={g('sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active'):.0f}% dram={(dr+dw)*sc/1e9:.2f}GB lanes={g('smsp__thread_inst_executed_per_inst_executed.ratio'):.1f} stalls={' '.join(f'{k}:{v:.1f}' for v,k in st)}")
