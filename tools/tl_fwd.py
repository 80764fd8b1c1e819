import numpy as np, sys
t=np.load(sys.argv[1] if len(sys.argv)>1 else 'gpurun_out/timeline_fwd.npy').astype(np.int64)
base=t[t>0].min(); t=np.where(t>0,t-base,-1)
n=(t[0,:,0]>=0).sum(); s=slice(10,n-1)
med=lambda x: float(np.median(x[s]))
print('kv tiles',n,'period', np.diff(t[0,10:n,0]).mean())
print('MMA: start->PV0 issued',med(t[0,:n,1]-t[0,:n,0]),'->S0 issued',med(t[0,:n,2]-t[0,:n,1]),'->PV1 issued',med(t[0,:n,3]-t[0,:n,2]),'->S1 issued',med(t[0,:n,4]-t[0,:n,3]),'-> next start',med(np.r_[t[0,1:n,0]-t[0,:n-1,4],0]))
for r in (1,2):
    sm=t[r,:n,1]-t[r,:n,0]; w=np.r_[t[r,1:n,0]-t[r,:n-1,1],0]
    print('softmax WG',r-1,'phase',med(sm),'wait next S',med(w))
#print('TMA K issue -> S0 issue', med(t[0,:n,2]-t[3,:n,0]))
for j in range(100,103): print(j, t[0,j,:5], t[1,j,:2], t[2,j,:2], t[3,j,0])
