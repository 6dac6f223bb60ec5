"""Accuracy check (CPU, exact FMA emulation via fractions) of the device exp used by
the spray source (fv2d_kernels.cuh: exp_estrin): worst relative error vs 60-digit
decimal over [-700, 700]; reports about 2 eps."""
from fractions import Fraction as F
import math, random
def fma(a,b,c): return float(F(a)*F(b)+F(c))
LOG2E=1.4426950408889634
LN2_HI=0.6931471805599453   # float(ln2)
LN2_LO=float(F(math.log(2)) - F(LN2_HI))  # placeholder; computed precisely below
import decimal
decimal.getcontext().prec=60
ln2=decimal.Decimal(2).ln()
LN2_HI=float(ln2)
LN2_LO=float(ln2-decimal.Decimal(LN2_HI))
C=[1.0/math.factorial(k) for k in range(13)]
def myexp(x):
    if x < -708.0: return 0.0
    if x > 709.0: return float('inf')
    t=x*LOG2E
    kd=(t+6755399441055744.0)-6755399441055744.0
    r=fma(kd,-LN2_HI,x); r=fma(kd,-LN2_LO,r)
    r2=r*r; r4=r2*r2; r8=r4*r4
    a0=fma(C[1],r,C[0]); a1=fma(C[3],r,C[2]); a2=fma(C[5],r,C[4]); a3=fma(C[7],r,C[6]); a4=fma(C[9],r,C[8]); a5=fma(C[11],r,C[10])
    b0=fma(a1,r2,a0); b1=fma(a3,r2,a2); b2=fma(a5,r2,a4); b3=C[12]
    c0=fma(b1,r4,b0); c1=fma(b3,r4,b2)
    p=fma(c1,r8,c0)
    k=int(kd)
    return math.ldexp(p,k)
random.seed(1); worst=0
for i in range(20000):
    x=random.uniform(-40,40) if i%2 else random.uniform(-700,700)
    y=myexp(x); ex=decimal.Decimal(x).exp()
    err=abs((decimal.Decimal(y)-ex)/ex)
    ulp=float(err)/2.220446049250313e-16
    worst=max(worst,ulp)
print("LN2_LO",repr(LN2_LO),"worst ulp (rel err / eps):",worst)

# exp_tab (FV2D_EXP_TAB): 2^k * 2^(j/64) * e^r, |r| <= ln2/128, degree-5 Estrin
x64 = decimal.Decimal(64) / ln2
C64 = float(x64)
L1 = float(ln2 / 64)
L2 = float(ln2 / 64 - decimal.Decimal(L1))
TAB = [float(decimal.Decimal(2) ** (decimal.Decimal(j) / 64)) for j in range(64)]
def exptab(x):
    if x > 709.0: return float('inf')
    tm = fma(x, C64, 6755399441055744.0)
    nd = tm - 6755399441055744.0
    n = int(nd)
    r = fma(nd, -L1, x); r = fma(nd, -L2, r)
    r2 = r * r
    a0 = r + 1.0
    a1 = fma(r, 1.0 / 6.0, 0.5)
    a2 = fma(r, 1.0 / 120.0, 1.0 / 24.0)
    b0 = fma(a1, r2, a0)
    r4 = r2 * r2
    p = fma(a2, r4, b0)
    k = max(min(n >> 6, 1023), -1022)
    return p * math.ldexp(TAB[n & 63], k)
random.seed(2); worst = 0
for i in range(20000):
    x = random.uniform(-40, 40) if i % 2 else random.uniform(-700, 700)
    y = exptab(x); ex = decimal.Decimal(x).exp()
    worst = max(worst, float(abs((decimal.Decimal(y) - ex) / ex)) / 2.220446049250313e-16)
print("exp_tab: C64", repr(C64), "L1", repr(L1), "L2", repr(L2), "worst ulp (rel err / eps):", worst)
