import csv,re,collections,sys,subprocess
rep, kname = sys.argv[1], sys.argv[2]
txt=open('/tmp/all.sass').read().split('\n')
# find section for kernel
start=[i for i,l in enumerate(txt) if l.startswith('//----') and kname in l][0]
end=next((i for i in range(start+1,len(txt)) if txt[i].startswith('//----')),len(txt))
cur=None; m={}
for L in txt[start:end]:
    mm=re.search(r'## File "([^"]+)", line (\d+)',L)
    if mm: cur=(mm.group(1).split('/')[-1],int(mm.group(2))); continue
    mo=re.search(r'/\*([0-9a-f]{4,})\*/',L)
    if mo: m[int(mo.group(1),16)]=cur
out=subprocess.run(['ncu','-i',rep,'--page','source','--csv','--print-source','sass'],capture_output=True,text=True).stdout
rows=list(csv.reader(out.splitlines())); h=rows[1]
iw=h.index('L1 Wavefronts Shared'); ie=h.index('Instructions Executed'); ix=h.index('L1 Wavefronts Shared Excessive'); isa=h.index('Warp Stall Sampling (All Samples)')
base=int(rows[2][0],16)
agg=collections.defaultdict(lambda:[0,0,0,0]); ops=collections.defaultdict(lambda:[0,0])
for r in rows[2:]:
    if len(r)<len(h): continue
    off=int(r[0],16)-base; k=m.get(off,('?',0))
    a=agg[k]; a[0]+=float(r[iw] or 0); a[1]+=float(r[ix] or 0); a[2]+=float(r[ie] or 0); a[3]+=float(r[isa] or 0)
    op=r[1].split(); op=[x for x in op if not x.startswith('@')]
    if op: o=ops[op[0].split('.')[0]]; o[0]+=float(r[ie] or 0); o[1]+=float(r[iw] or 0)
N=65536; ts=sum(a[3] for a in agg.values())
print('total wf/mat %.0f ins/mat %.0f'%(sum(a[0] for a in agg.values())/N, sum(a[2] for a in agg.values())/N))
src={}
for f in ['batched64.cuh','batched.cu']:
    src[f]=open('/root/repo/paper_0901_1696_b200/csrc/'+f).read().split('\n')
print('wf/mat exc/mat ins/mat samp%')
for k,a in sorted(agg.items(),key=lambda x:-x[1][0])[:int(sys.argv[3]) if len(sys.argv)>3 else 25]:
    s=src[k[0]][k[1]-1].strip()[:70] if k[0] in src else ''
    print('%7.0f %6.0f %6.0f %5.1f %s:%d %s'%(a[0]/N,a[1]/N,a[2]/N,100*a[3]/ts,k[0],k[1],s))
print('--- by samples')
for k,a in sorted(agg.items(),key=lambda x:-x[1][3])[:20]:
    s=src[k[0]][k[1]-1].strip()[:70] if k[0] in src else ''
    print('%7.0f %6.0f %6.0f %5.1f %s:%d %s'%(a[0]/N,a[1]/N,a[2]/N,100*a[3]/ts,k[0],k[1],s))
print('--- ops')
for k,v in sorted(ops.items(),key=lambda x:-x[1][0])[:16]: print('%-8s ins/mat %6.0f wf/mat %6.0f'%(k,v[0]/N,v[1]/N))
