import numpy as np, torch, sys
sys.path.insert(0, '.')
from oracle.oracle import Rng, random_field
from paper_2301_11828_b200.engine import FastForce, build_kernel
from paper_2301_11828_b200.slab import SlabForce
dev = torch.device("cuda:0")
dims=(256,256); M=3; n=256*256; h=1/256
K = build_kernel(2, h, 3.015*h, M, 1.0, 1.0)
u = torch.from_numpy(np.stack([random_field(Rng(4200 + i), 2, n) for i in range(2)])).to(dev)
full = FastForce(dims, M, K); f_ref = torch.zeros_like(u)
full.matvec_device(u, f_ref, 2, stream=torch.cuda.current_stream()); torch.cuda.synchronize()
for r in range(4):
    sf = SlabForce(dims, M, K, rank=r, world=4, device=dev)
    lo=(sf.r0-sf.gl)*256; hi=(sf.r1+sf.gh)*256
    ext_u = u[:, :, lo:hi].contiguous()
    fe = torch.zeros_like(ext_u)
    sf.eng.matvec_device(ext_u, fe, 2, stream=torch.cuda.current_stream()); torch.cuda.synchronize()
    ref = f_ref[:, :, lo:hi]
    d = (fe-ref).abs().reshape(2,2,-1,256).amax(dim=(0,1,3))
    print(r, sf.r0, sf.r1, sf.gl, sf.gh, 'row maxerr:', [f"{x:.1e}" for x in d.tolist()][:8], '...', [f"{x:.1e}" for x in d.tolist()][-8:])
    # also apply only
    fa = torch.zeros_like(ext_u); sf.eng.apply_device(ext_u, fa, 2, stream=torch.cuda.current_stream())
    fr = torch.zeros_like(u); full.apply_device(u, fr, 2, stream=torch.cuda.current_stream()); torch.cuda.synchronize()
    da = (fa-fr[:, :, lo:hi]).abs().reshape(2,2,-1,256).amax(dim=(0,1,3))
    print('   apply row maxerr', [f"{x:.1e}" for x in da.tolist()][:8], [f"{x:.1e}" for x in da.tolist()][-8:])
