"""Remez fits of the sin / cos kernels on |y| <= pi/4 in 50-digit arithmetic (dev tool):
prints the coefficients and max absolute error for 6, 5 and 4 coefficients.
kernels.cuh uses the 5-coefficient cos fit (kCos5)."""
import mpmath as mp
mp.mp.dps = 50
T = (mp.pi/4)**2
def fit(fun, w, nc, npts=400):
    # weighted least squares on Chebyshev nodes in t in (0, T], then Remez iterations
    import itertools
    nodes=[T*(1-mp.cos(mp.pi*(k+0.5)/npts))/2 for k in range(npts)]
    # Remez: start with Chebyshev extrema
    m=nc+1
    xs=[T*(1-mp.cos(mp.pi*k/(m-1)))/2 for k in range(m)]
    xs[0]=T*mp.mpf('1e-6')
    for it in range(30):
        # solve sum c_j t^j * w(t) + (-1)^i E = fun(t)*w(t)... we approximate g(t)=fun(t) by poly with weight w
        A=mp.matrix(m,m); b=mp.matrix(m,1)
        for i,t in enumerate(xs):
            for j in range(nc): A[i,j]=w(t)*t**j
            A[i,nc]=(-1)**i
            b[i]=w(t)*fun(t)
        sol=mp.lu_solve(A,b)
        c=[sol[j] for j in range(nc)]; E=sol[nc]
        err=lambda t: w(t)*(fun(t)-sum(c[j]*t**j for j in range(nc)))
        # find extrema on a fine grid
        grid=[T*k/4000 for k in range(1,4001)]
        vals=[err(t) for t in grid]
        ext=[]
        for k in range(len(grid)):
            left=vals[k-1] if k>0 else None; right=vals[k+1] if k<len(grid)-1 else None
            v=vals[k]
            if (left is None or abs(v)>=abs(left)) and (right is None or abs(v)>=abs(right)): ext.append((grid[k],v))
        # keep alternating extrema: choose m largest with alternating signs
        # simple approach: merge by sign groups
        groups=[]
        for t,v in [(g,vv) for g,vv in zip(grid,vals)]:
            s=1 if v>=0 else -1
            if groups and groups[-1][0]==s:
                if abs(v)>abs(groups[-1][2]): groups[-1]=(s,t,v)
            else: groups.append((s,t,v))
        if len(groups)>=m:
            # pick m consecutive groups with the largest minimum
            best=None
            for st in range(len(groups)-m+1):
                mn=min(abs(g[2]) for g in groups[st:st+m])
                if best is None or mn>best[0]: best=(mn,st)
            xs=[g[1] for g in groups[best[1]:best[1]+m]]
        maxerr=max(abs(v) for v in vals)
    return c, maxerr
# cos(y) = 1 - t/2 + t^2 Q(t): Q(t) = (cos(sqrt t) - 1 + t/2)/t^2, absolute error weight t^2
fc=lambda t: (mp.cos(mp.sqrt(t))-1+t/2)/t**2
for nc in (6,5,4):
    c,e=fit(fc, lambda t: t**2, nc)
    print('cos nc',nc,'max abs err %.3e'%float(e), [mp.nstr(x,20) for x in c[::-1]])
# sin(y) = y + y^3 P(t): P(t) = (sin(sqrt t)/sqrt t - 1)/t, abs error weight y^3 = t^1.5
fs=lambda t: (mp.sin(mp.sqrt(t))/mp.sqrt(t)-1)/t
for nc in (6,5,4):
    c,e=fit(fs, lambda t: t**mp.mpf(1.5), nc)
    print('sin nc',nc,'max abs err %.3e'%float(e), [mp.nstr(x,20) for x in c[::-1]])
