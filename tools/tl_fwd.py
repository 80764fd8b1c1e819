import numpy as np, sys
t=np.load(sys.argv[1] if len(sys.argv)>1 else 'gpurun_out/timeline_fwd.npy').astype(np.int64)
base=t[t>0].min(); t=np.where(t>0,t-base,-1)
n=(t[0,:,0]>=0).sum(); s=slice(10,n-1)
med=lambda x: float(np.median(x[s]))
print('kv tiles',n,'period', np.diff(t[0,10:n,0]).mean())
print('MMA: start->PV0 issued',med(t[0,:n,1]-t[0,:n,0]),'->S0 issued',med(t[0,:n,2]-t[0,:n,1]),'->PV1 issued',med(t[0,:n,3]-t[0,:n,2]),'->S1 issued',med(t[0,:n,4]-t[0,:n,3]),'-> next start',med(np.r_[t[0,1:n,0]-t[0,:n-1,4],0]))
for r in (1,2):
    sm=t[r,:n,1]-t[r,:n,0]; w=np.r_[t[r,1:n,0]-t[r,:n-1,1],0]
    print('softmax WG',r-1,'phase',med(sm),'(ld',med(t[r,:n,2]-t[r,:n,0]),'max',med(t[r,:n,3]-t[r,:n,2]),'exp',med(t[r,:n,1]-t[r,:n,3]),') wait next S',med(w))
    # S_t(j) issued (MMA stamp) -> softmax sees S
    print('   S issue -> seen', med(t[r,:n,0]-t[0,:n,2*r]), ' P arrive -> PV issued(next j)', med(t[0,1:n+1,2*r-1][:n]-t[r,:n,1]) if n+1<=t.shape[1] else '')
