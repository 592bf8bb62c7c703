import json, sys
s = json.load(open(sys.argv[1]))
ops = s["ops"]
tp = s["tp"]; cfg0 = s["cfg0"]; tiles = sorted(s["tile"])
def nib(c, j): return (c >> (4*j)) & 15
L = []
E = L.append
E('#include <cstdint>')
E('struct __align__(16) P_t { unsigned long long rank_bits; double m[%d][8]; };' % len(ops))
E('__device__ __forceinline__ unsigned long long iz(unsigned long long v, int p){return ((v>>p)<<(p+1))|(v&((1ULL<<p)-1));}')
E('__device__ __forceinline__ int swz(int s){return s ^ (((s>>3)^(s>>6)^(s>>9))&7);}')
E('extern "C" __global__ void __launch_bounds__(256,2) kpass(const __grid_constant__ P_t P, double2* __restrict__ st){')
E(' extern __shared__ double2 sm[];')
E(' const int lane=threadIdx.x&31, warp=threadIdx.x>>5;')
E(' unsigned long long base=blockIdx.x;')
for t in tiles: E(' base=iz(base,%d);' % t)
E(' const unsigned long long gcta = P.rank_bits | base;')
names = [f"a{i}" for i in range(16)]
E(' double2 ' + ','.join(names) + ';')
def gcoords(c):
    # global lane/warp offset expr
    terms = ['((unsigned long long)((lane&3)<<1))']
    for j in range(2,5): terms.append(f'((unsigned long long)((lane>>{j})&1)<<{tp[nib(c,4+j)]})')
    for j in range(3): terms.append(f'((unsigned long long)((warp>>{j})&1)<<{tp[nib(c,9+j)]})')
    return '|'.join(terms)
cur = cfg0
reg = list(range(16))  # logical register i -> variable index
E(' { const double2* p = st + base + (%s);' % gcoords(cur))
for j in range(8):
    off = sum(((j>>b)&1) << tp[nib(cur,1+b)] for b in range(3))
    E(f'  {{ double x0,x1,x2,x3; asm volatile("ld.global.v4.f64 {{%0,%1,%2,%3}}, [%4];" : "=d"(x0),"=d"(x1),"=d"(x2),"=d"(x3) : "l"(p+{off}ULL)); a{2*j}=make_double2(x0,x1); a{2*j+1}=make_double2(x2,x3);}}')
E(' }')
def scoords(c, tag):
    st = ' | '.join([f'(((lane>>{j})&1)<<{nib(c,4+j)})' for j in range(5)] + [f'(((warp>>{j})&1)<<{nib(c,9+j)})' for j in range(3)])
    E(f'  const int zt{tag} = swz({st});')
    return [f'{(1<<nib(c,j)) ^ ((( (1<<nib(c,j))>>3) ^ ((1<<nib(c,j))>>6) ^ ((1<<nib(c,j))>>9))&7)}' for j in range(4)]
for o, op in enumerate(ops):
    code = op["code"]
    if code == 4:
        E(' {')
        zr = scoords(cur, 'a')
        for i in range(16):
            z = ' ^ '.join(['zta'] + [zr[b] for b in range(4) if (i>>b)&1])
            E(f'  sm[{z}] = a{reg[i]};')
        E('  __syncthreads();')
        cur = op["cfg"]
        zr = scoords(cur, 'b')
        for i in range(16):
            z = ' ^ '.join(['ztb'] + [zr[b] for b in range(4) if (i>>b)&1])
            E(f'  a{reg[i]} = sm[{z}];')
        E('  __syncthreads();')
        E(' }')
        continue
    pred = []
    if op["mlane"]: pred.append(f'((lane&{op["mlane"]})=={op["vlane"]})')
    if op["mwarp"]: pred.append(f'((warp&{op["mwarp"]})=={op["vwarp"]})')
    if op["mout"]: pred.append(f'((gcta&{op["mout"]}ULL)=={op["vout"]}ULL)')
    E(' { const bool tp = %s;' % (' && '.join(pred) if pred else 'true'))
    k = op["k"]; mreg = op["mreg"]; vreg = op["vreg"]
    if code == 3:
        for i in range(16):
            if (i & mreg) != vreg: continue
            v = f'a{reg[i]}'
            E(f'  {{ const double p1=-P.m[{o}][1]*{v}.y, p2=P.m[{o}][1]*{v}.x; const double nx=fma(P.m[{o}][0],{v}.x,p1), ny=fma(P.m[{o}][0],{v}.y,p2); {v}.x=tp?nx:{v}.x; {v}.y=tp?ny:{v}.y; }}')
    else:
        for p in range(8):
            i0 = ((p >> k) << (k+1)) | (p & ((1<<k)-1)); i1 = i0 | (1<<k)
            if (i0 & mreg) != vreg: continue
            x, y = f'a{reg[i0]}', f'a{reg[i1]}'
            if code == 2:
                if pred:
                    E(f'  {{ const double2 t={x}; {x}.x=tp?{y}.x:{x}.x; {x}.y=tp?{y}.y:{x}.y; {y}.x=tp?t.x:{y}.x; {y}.y=tp?t.y:{y}.y; }}')
                else:
                    reg[i0], reg[i1] = reg[i1], reg[i0]
            elif code == 1:
                m = f'P.m[{o}]'
                E(f'  {{ const double p1={m}[2]*{y}.x,p2={m}[2]*{y}.y,p3={m}[4]*{x}.x,p4={m}[4]*{x}.y; {x}.x=fma({m}[0],{x}.x,p1); {x}.y=fma({m}[0],{x}.y,p2); {y}.x=fma({m}[6],{y}.x,p3); {y}.y=fma({m}[6],{y}.y,p4); }}')
                if pred: raise SystemExit("pred U2R unsupported in prototype")
            else:
                if pred: raise SystemExit("pred U2 unsupported in prototype")
                m = f'P.m[{o}]'
                E(f'  {{ const double p1=fma(-{m}[1],{x}.y,fma({m}[2],{y}.x,-{m}[3]*{y}.y)); const double p2=fma({m}[1],{x}.x,fma({m}[2],{y}.y,{m}[3]*{y}.x)); const double p3=fma({m}[4],{x}.x,fma(-{m}[5],{x}.y,-{m}[7]*{y}.y)); const double p4=fma({m}[4],{x}.y,fma({m}[5],{x}.x,{m}[7]*{y}.x)); {x}.x=fma({m}[0],{x}.x,p1); {x}.y=fma({m}[0],{x}.y,p2); {y}.x=fma({m}[6],{y}.x,p3); {y}.y=fma({m}[6],{y}.y,p4); }}')
    E(' }')
E(' { double2* p = st + base + (%s);' % gcoords(cur))
for j in range(8):
    off = sum(((j>>b)&1) << tp[nib(cur,1+b)] for b in range(3))
    E(f'  asm volatile("st.global.v4.f64 [%0], {{%1,%2,%3,%4}};" :: "l"(p+{off}ULL), "d"(a{reg[2*j]}.x),"d"(a{reg[2*j]}.y),"d"(a{reg[2*j+1]}.x),"d"(a{reg[2*j+1]}.y) : "memory");')
E(' }')
E('}')
open(sys.argv[2],'w').write('\n'.join(L))
