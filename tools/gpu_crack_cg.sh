mkdir -p gpurun_out
timeout 600 python tools/crack_scan.py > gpurun_out/crack_scan.log 2>&1
timeout 300 python tools/cg_iter.py > gpurun_out/cg_iter.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/cg1_launches.csv python -c "
import sys,torch; sys.path.insert(0,'.')
from paper_2301_11828_b200 import FastForce, build_kernel
n=128; h=1/n; dl=3.015*h
ff=FastForce((n,n),3,build_kernel(2,h,dl,3,1.0,1.0),device=0); ff.set_geometry(h,[0,0],dl,1.0)
for ax in range(2):
    lo=[-9,-9]; hi=[9,9]; hi[ax]=dl; ff.add_constraint(lo,hi,3,0,0.0)
    lo=[-9,-9]; hi=[9,9]; lo[ax]=1-dl; ff.add_constraint(lo,hi,3,0,0.0)
b=torch.empty((2,n*n),dtype=torch.float64,device='cuda').uniform_(-1,1); x=torch.empty_like(b)
ff.cg_solve_device(b,x,tol=1e-30,maxit=5)
" > gpurun_out/cg1_ncu.log 2>&1
echo done
