import csv, re, sys
def load(path):
    rows=[r for r in csv.reader(l for l in open(path) if not l.startswith('=='))]
    h=rows[0]; ix={k:i for i,k in enumerate(h)}
    L={}; order=[]
    for r in rows[1:]:
        if len(r)<len(h): continue
        k=r[ix['ID']]
        if k not in L: L[k]={}; order.append(k)
        v=float(r[ix['Metric Value']].replace(',',''))
        L[k][r[ix['Metric Name']]]=v
    return [L[k] for k in order]
for p in sys.argv[1:]:
    ls=load(p)
    print(p, len(ls))
    for i in (0,8,16,24,32):
        if i>=len(ls): continue
        a=ls[i]
        rd=a['lts__t_sectors_op_read.sum']*32/1e9; hit=a['lts__t_sectors_op_read_lookup_hit.sum']/max(a['lts__t_sectors_op_read.sum'],1)
        print(f"  size#{i}: {a['gpu__time_duration.sum']/1e6:.2f} ms dram_rd {a['dram__bytes_read.sum']/1e9:.1f} GB  L2 rd {rd:.1f} GB hit {hit:.2%} miss {a['lts__t_sectors_op_read_lookup_miss.sum']*32/1e9:.1f} GB")
    print('  total ms', sum(a['gpu__time_duration.sum'] for a in ls)/1e6, 'dram GB', sum(a['dram__bytes_read.sum'] for a in ls)/1e9)
