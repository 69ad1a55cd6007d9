import sys, numpy as np, torch
sys.path.insert(0,'.'); sys.path.insert(0,'oracle')
import flashmp_oracle as O
from paper_2508_07193_b200 import _lib
from paper_2508_07193_b200.plan import SolvePlan, SubSpec, block_struct
for dims in [(1,1,1),(2,2,2),(4,5,6)]:
    alpha=0.25
    od=O.precompute(dims,alpha)
    dof=3*int(np.prod(dims))
    r=np.random.default_rng(0).uniform(-1,1,dof)
    e0=O.exact_solve(dims,od.binv,r)
    plan=SolvePlan([SubSpec(dims,(0,0,0),(0,0,0),dims)],alpha,'cuda',need_woodbury=False)
    R=torch.from_numpy(r).cuda()
    plan.apply(block_struct(*dims),_lib.FMP_SOLVE_FACES,R,None)
    Y=plan.ymat[0][0].cpu().numpy()
    print(dims,'faces err',np.abs(Y-e0[od.rows]).max())
    cinv=torch.from_numpy(od.Cinv.copy()).cuda()
    plan2=SolvePlan([SubSpec(dims,(0,0,0),(0,0,0),dims)],alpha,'cuda',cinv={dims:cinv})
    Z=torch.empty_like(R)
    plan2.apply(block_struct(*dims),_lib.FMP_SOLVE_WOODBURY,R,Z)
    torch.cuda.synchronize()
    print(' Y2 err',np.abs(plan2.ymat[0][0].cpu().numpy()-e0[od.rows]).max(),
          ' Z err',np.abs(plan2.zmat[0][0].cpu().numpy()-od.Cinv@e0[od.rows]).max(),
          ' solve err',np.abs(Z.cpu().numpy()-O.solve(od,r)).max())
