"""Search XOR swizzles (bijective: the XOR term reads bits >= 3 only) for the 512/1024-point
line kernels (python3 tools/layouts/search_line_swizzle.py)."""
import math, itertools
exec(open(__file__.replace('search_line_swizzle.py', 'bank_conflicts.py')).read().split('for H in (128,256,512):')[0])
def cost_lines(n, pos):  # pos(l, p) -> element index
    P,R,T=plan(n); TM=max(T); L=256//TM
    R0,R1=R[0],R[1]; T0,T1=T[0],T[1]
    def p0out(e): return (e%T1)*R1 + e//T1
    def p1(i,r): return i*R1+r
    def p2in(e):
        i1=(e//(R0*R1))*R0 + e%R0; r1=(e//R0)%R1; return i1*R1+r1
    tot=0; per={}
    for name in ["p0st","p1","last"]:
        c0=tot
        for w in range(8):
            for r in range(max(R)):
                ad=[]
                for t in range(w*32,w*32+32):
                    l=t%L; i=t//L
                    if name=="p0st": q=p0out(i*R0+r) if (i<T0 and r<R0) else None
                    elif name=="p1": q=p1(i,r) if (P==3 and i<T1 and r<R1) else None
                    else:
                        RLs=R[-1]; TLs=n//RLs
                        q=(p1(i,r) if P==2 else p2in(i+r*TLs)) if (r<RLs and i<TLs) else None
                    ad.append(None if q is None else pos(l,q))
                tot+=wavefronts(ad)
        per[name]=tot-c0
    return tot, per
for n in (512,1024,256):
    P,R,T=plan(n); L=256//max(T)
    best=[]
    for a,b,s in itertools.product(range(0,10),range(0,10),range(0,8)):
        if b<a: continue
        def pos(l,p,a=a,b=b,s=s,n=n):
            x=((p>>a)^(p>>b) if b!=a else (p>>a))
            return l*n + (p ^ ((x + s*l) & 7))
        if len({pos(0,p) for p in range(n)})<n or len({pos(1,p) for p in range(n)})<n: continue
        c,per=cost_lines(n,pos)
        best.append((c,a,b,s,per))
    best.sort(key=lambda x:x[0])
    print(n, "L",L, best[:4])
