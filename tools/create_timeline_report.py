"""Diagnostics: per-product DMMA rate and GPU utilisation over one gls_create, from the files
tools/create_timeline.py writes (run it with GLS_TRACE_GEMM=1, stderr -> gpurun_out/tl_gemm.log).
Matches every [gemm] line (shape, triangular flags, stream) to its kernel record, counts the flops the
triangular flags leave, and prints the products above 2 GFLOP with their TF/s plus a 0.25 ms
utilisation timeline.  usage: python tools/create_timeline_report.py [n]"""
import json, collections, numpy as np, re
import sys
n = sys.argv[1] if len(sys.argv) > 1 else "10000"
d=json.load(open("gpurun_out/create_timeline_n%s.json" % n))
lines=[l for l in open('gpurun_out/tl_gemm.log') if l.startswith('[gemm]')]
per=len(lines)//4; lines=lines[-per:]
calls=collections.defaultdict(list)
for l in lines:
    f=l.split(); M,N,K=int(f[1]),int(f[2]),int(f[3]); op=f[4]; fl=int(f[6]); st=f[8]; cap=int(f[10])
    calls[st].append((M,N,K,op,fl,cap))
def isg(nm): return any(k in nm for k in ['dgemm_tma_kernel','dgemm_small_kernel','dgemm_kernel'])
ks=collections.defaultdict(list)
for r in d:
    if isg(r[0]): ks[r[1]].append(r)
cnt_calls={k:len(v) for k,v in calls.items()}; cnt_ks={k:len(v) for k,v in ks.items()}
print(sorted(cnt_calls.values()), sorted(cnt_ks.values()))
def fma(M,N,K,fl):
    r=np.arange(0,M,16)+8; c=np.arange(0,N,16)+8
    R,C=np.meshgrid(r,c,indexing='ij')
    kb=np.where(fl&4, C, 0); ke=np.full(R.shape,K)
    if fl&2: ke=np.minimum(ke,C+1)
    if fl&1: ke=np.minimum(ke,R+1)
    L=np.maximum(ke-kb,0).astype(float)
    if fl&8: L=np.where(C>R,0,L)
    return L.sum()*256
# match streams by count
used=set(); res=[]
for sp,cl in calls.items():
    cands=[k for k,v in ks.items() if len(v)==len(cl) and k not in used]
    if not cands: print('nomatch',sp,len(cl)); continue
    k=cands[0]; used.add(k)
    for c,kr in zip(cl,ks[k]):
        f=2*fma(c[0],c[1],c[2],c[4]); res.append((kr[2],kr[3],f,c,kr[0][:20],k))
t0=d[0][2]
tot=sum(r[2] for r in res); print('total gemm flop %.3e'%tot)
res.sort()
big=[r for r in res if r[2]>2e9]
for r in big: print('t=%7.2f dur=%7.1fus %6.1f TF/s %s %s st%s'%((r[0]-t0)/1e3,r[1],r[2]/r[1]/1e6,r[3],r[4],r[5]))
small=[r for r in res if r[2]<=2e9]
print('small gemms', len(small), 'sum dur %.2f ms'%(sum(r[1] for r in small)/1e3), 'flop %.3e'%sum(r[2] for r in small))
# utilization timeline in 0.5 ms bins
import math
t1=max(r[0]+r[1] for r in res); span=(t1-t0)
bins=np.zeros(int(math.ceil(span/250))+1)
for ts,du,f,c,nm,st in res:
    a=(ts-t0)/250; b=(ts+du-t0)/250; rate=f/du  # flop per us
    i=int(a)
    while i<b:
        lo=max(a,i); hi=min(b,i+1); bins[i]+=rate*(hi-lo)*250; i+=1
print('TF/s per 0.25ms bin:'); print(' '.join('%d'%(v/250/1e6) for v in bins))
print('time below 20 TF/s: %.2f ms'%(0.25*np.sum(bins/250/1e6<20)))
