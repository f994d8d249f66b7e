# complex64 design check (DESIGN 3.4): can fp32-arithmetic fine-level Vanka sweeps reach relres 1e-5 at h = 1/1024
# (C4 set A, slot 0), with the convergence and restricted residuals formed in fp64 from the fp32-stored iterate?
# numpy emulation of V(1,1); coarse levels fp64.  Modes: fp32sweep (all sweep arithmetic fp32), fp32vanka (fp64
# residual, fp32 Vanka stencil), fp64sweep (fp32 storage, fp64 arithmetic: the shipped design).
#   python tools/c64_fp32_emulation.py 1024 fp32sweep   -> stalls at 1.17e-5
#   python tools/c64_fp32_emulation.py 1024 fp32vanka   -> 9.8e-6 after 11 cycles
#   python tools/c64_fp32_emulation.py 1024 fp64sweep   -> 7.1e-6 after 6 cycles
import numpy as np, sys
sys.path.insert(0, __import__('os').path.join(__import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))), 'tests'))
from oracle_lib import Oracle
O = Oracle()
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
mode = sys.argv[2] if len(sys.argv) > 2 else 'fp32sweep'
m = n - 1
lam = O.circulant_shifts(0.01, 1024, 1/1024, 0, 1)[0]
b = O.random_complex(3, m*m).reshape(m, m)
omega = 24/25
def vanka(eta):
    i2, i4, i6 = 1/(2+eta), 1/(4+eta), 1/(6+eta)
    return 0.25*(i2+2*i4+i6), 0.25*(i2-i6), 0.25*(i2-2*i4+i6)
def pad(x): return np.pad(x, 1)
def Lop(u, n, dt):
    h2 = (1.0/n)**2; z = pad(u)
    eta = dt(lam*h2)
    return ((dt(4)+eta)*z[1:-1,1:-1] - z[:-2,1:-1] - z[2:,1:-1] - z[1:-1,:-2] - z[1:-1,2:]) / dt(h2)
def smooth(u, b, n, dt):
    h = 1.0/n; eta = lam*h*h
    a, bb, c = vanka(eta)
    k0, k1, k2 = [dt(omega*h*h/4*x) for x in (4*a, 2*bb, c)]
    if mode == 'fp32vanka' and dt == np.complex64:
        r = (b - Lop(u.astype(np.complex128), n, np.complex128)).astype(np.complex64)
    else:
        r = b.astype(dt) - Lop(u.astype(dt), n, dt)
    z = pad(r)
    s_e = z[1:-1,:-2]+z[1:-1,2:]+z[:-2,1:-1]+z[2:,1:-1]
    s_c = z[:-2,:-2]+z[:-2,2:]+z[2:,:-2]+z[2:,2:]
    return (u.astype(dt) + k0*r + k1*s_e + k2*s_c)
def R(f):
    mc = (f.shape[0]-1)//2
    z = pad(f)
    out = np.zeros((mc,mc), f.dtype)
    c = z[2:-1:2,2:-1:2]
    out = (4*z[2:2*mc+1:2,2:2*mc+1:2] + 2*(z[1:2*mc:2,2:2*mc+1:2]+z[3:2*mc+2:2,2:2*mc+1:2]+z[2:2*mc+1:2,1:2*mc:2]+z[2:2*mc+1:2,3:2*mc+2:2])
           + z[1:2*mc:2,1:2*mc:2]+z[1:2*mc:2,3:2*mc+2:2]+z[3:2*mc+2:2,1:2*mc:2]+z[3:2*mc+2:2,3:2*mc+2:2])/16
    return out
def Pr(e, mf):
    z = pad(e); out = np.zeros((mf,mf), e.dtype)
    out[1::2,1::2] = e
    out[0::2,1::2] = 0.5*(z[:-1,1:-1]+z[1:,1:-1])
    out[1::2,0::2] = 0.5*(z[1:-1,:-1]+z[1:-1,1:])
    out[0::2,0::2] = 0.25*(z[:-1,:-1]+z[1:,:-1]+z[:-1,1:]+z[1:,1:])
    return out
def vcycle(u, b, n, fine):
    if n == 4:
        # direct solve 3x3
        A = O.dense_operator(4, lam); return np.linalg.solve(A, b.ravel()).reshape(3,3)
    dt = np.complex64 if (fine and mode in ('fp32sweep', 'fp32vanka')) else np.complex128
    u = smooth(u, b, n, dt)
    if fine: u = u.astype(np.complex64).astype(np.complex128)
    else: u = u.astype(np.complex128)
    r = b - Lop(u, n, np.complex128)
    rc = R(r)
    ec = vcycle(np.zeros_like(rc), rc, n//2, False)
    u = u + Pr(ec, n-1)
    if fine: u = u.astype(np.complex64).astype(np.complex128)
    u = smooth(u, b, n, dt)
    if fine: u = u.astype(np.complex64).astype(np.complex128)
    return u.astype(np.complex128)
u = np.zeros((m,m), np.complex128)
r0 = np.linalg.norm(b)
for k in range(1, 30):
    u = vcycle(u, b, n, True)
    rr = np.linalg.norm(b - Lop(u, n, np.complex128)) / r0
    print(k, f"{rr:.3e}", flush=True)
    if rr <= 1e-5: break
