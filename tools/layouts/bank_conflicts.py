"""Quarter-warp bank-group model of the shared-memory accesses of the row C2R (row-major
thread mapping) and line kernels (line-fastest mapping) of fw_lines.cu: wavefronts per pass for
candidate paddings (python3 tools/layouts/bank_conflicts.py)."""
import math
def ilog2(n): return n.bit_length()-1
def npass(n): return (ilog2(n)+3)//4
def radix(n,i):
    L=ilog2(n); P=npass(n); return 1<<(L//P + (1 if i < L%P else 0))
def plan(H):
    P=npass(H); R=[radix(H,i) for i in range(P)]; T=[H//r for r in R]
    return P,R,T
def wavefronts(addrs):  # list of 32 element indices (16B each) or None; quarter-warp phases
    tot=0
    for q in range(4):
        grp={}
        for a in addrs[q*8:(q+1)*8]:
            if a is None: continue
            grp.setdefault(a%8,set()).add(a)
        tot+= max([len(v) for v in grp.values()] or [0])
    return tot
def analyze(H, pad, LS, label):
    P,R,T=plan(H); TM=max(T); TL=T[-1]
    R0,R1=R[0],R[1]; T0,T1=T[0],T[1]
    S1=ilog2(R1); ST=ilog2(T1)
    def p0out(e): return pad((e%T1)*R1 + e//T1)
    def p1(i,r): return pad(i*R1+r)
    def p2in(e):
        i1=(e//(R0*R1))*R0 + e%R0; r1=(e//R0)%R1; return pad(i1*R1+r1)
    res={}
    nthreads=256 if TM<=256 else TM
    for name in ["p0st","p1","last"]:
        tot=0; ideal=0
        for w in range(0, 256//32 if TM<=32 else 8):
            tids=range(w*32,w*32+32)
            for r in range(max(R)):
                ad=[]
                for t in tids:
                    rl=t//TM; i=t%TM
                    base=rl*LS
                    if name=="p0st":
                        ad.append(base+p0out(i*R0+r) if (i<T0 and r<R0) else None)
                    elif name=="p1":
                        ad.append(base+p1(i,r) if (P==3 and i<T1 and r<R1) else None)
                    else:
                        RL=R[-1]
                        if r>=RL or i>=TL: ad.append(None)
                        else: ad.append(base+(p1(i,r) if P==2 else p2in(i+r*TL)))
                tot+=wavefronts(ad); ideal+=sum(math.ceil(sum(1 for a in ad[q*8:q*8+8] if a is not None)/8) for q in range(4))
        res[name]=(tot,ideal)
    print(label, H, res)
for H in (128,256,512):
    P,R,T=plan(H); S1=ilog2(R[1]); ST=ilog2(T[1])
    cur=lambda p,S1=S1,ST=ST: p+(p>>S1)+(p>>ST)
    LS=((H-1)+((H-1)>>S1)+((H-1)>>ST)+1)|1
    analyze(H,cur,LS,"current")
    for sh in (2,3,4,5):
        f=lambda p,sh=sh: p+(p>>sh)
        LS2=((H-1)+((H-1)>>sh)+1)|1
        analyze(H,f,LS2,f"p+(p>>{sh})")

print("---- k_lines mapping (l = tid % L, i = tid / L), line stride LS")
def analyze_lines(n):
    P,R,T=plan(n); TM=max(T); L=256//TM
    R0,R1=R[0],R[1]; T0,T1=T[0],T[1]
    S1=ilog2(R1); ST=ilog2(T1)
    pad=lambda p: p+(p>>S1)+(p>>ST)
    LS=((n-1)+((n-1)>>S1)+((n-1)>>ST)+1)|1
    def p0out(e): return pad((e%T1)*R1 + e//T1)
    def p1(i,r): return pad(i*R1+r)
    def p2in(e):
        i1=(e//(R0*R1))*R0 + e%R0; r1=(e//R0)%R1; return pad(i1*R1+r1)
    res={}
    for name in ["p0st","p1","last"]:
        tot=0; ideal=0
        for w in range(8):
            for r in range(max(R)):
                ad=[]
                for t in range(w*32,w*32+32):
                    l=t%L; i=t//L; base=l*LS
                    if name=="p0st": ad.append(base+p0out(i*R0+r) if (i<T0 and r<R0) else None)
                    elif name=="p1": ad.append(base+p1(i,r) if (P==3 and i<T1 and r<R1) else None)
                    else:
                        RLs=R[-1]; TLs=n//RLs
                        ad.append(base+(p1(i,r) if P==2 else p2in(i+r*TLs)) if (r<RLs and i<TLs) else None)
                tot+=wavefronts(ad); ideal+=sum(math.ceil(sum(1 for a in ad[q*8:q*8+8] if a is not None)/8) for q in range(4))
        res[name]=(tot,ideal)
    print("k_lines", n, "L", L, res)
for n in (256,512,1024): analyze_lines(n)
