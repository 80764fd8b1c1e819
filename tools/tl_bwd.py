import numpy as np, sys
t=np.load(sys.argv[1] if len(sys.argv)>1 else 'gpurun_out/timeline_bwd.npy').astype(np.int64)
base=t[t>0].min(); t=np.where(t>0,t-base,-1)
n=(t[0,:,0]>=0).sum(); s=slice(10,n-1)
m=t[0,:n,0]; print('tiles',n,'period',np.diff(m[10:n]).mean())
med=lambda x: float(np.median(x[s]))
print('compute: P phase',med(t[1,:n,1]-t[1,:n,0]),'wait dP',med(t[1,:n,2]-t[1,:n,1]),'dS phase',med(t[1,:n,3]-t[1,:n,2]),'wait next S',med(np.r_[t[1,1:n,0]-t[1,:n-1,3],0]))
print('MMA: dP issue->P ready(dV)',med(t[0,:n,1]-t[0,:n,0]),'dV->S issued',med(t[0,:n,2]-t[0,:n,1]),'S issued->dS ready',med(t[0,:n,3]-t[0,:n,2]),'dQ/dK issue -> next dP issue',med(np.r_[t[0,1:n,0]-t[0,:n-1,3],0]))
print('drain: dQ issue->dQF',med(t[2,:n,0]-t[0,:n,3]),'dQF->DQE',med(t[2,:n,1]-t[2,:n,0]),'dQF->done',med(t[2,:n,2]-t[2,:n,0]))
