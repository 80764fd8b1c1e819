import numpy as np, sys
t=np.load(sys.argv[1]).astype(np.int64)
base=t[t>0].min(); t=np.where(t>0,t-base,-1)
n=(t[1,:,0]>=0).sum(); s=slice(10,n-2)
med=lambda x: float(np.median(x[s]))
print('tiles',n,'softmax0 period',np.diff(t[1,10:n,0]).mean(),'softmax1 period',np.diff(t[2,10:n,0]).mean())
for r in (1,2):
    print('WG',r-1,'ld',med(t[r,:n,1]-t[r,:n,0]),'max',med(t[r,:n,2]-t[r,:n,1]),'exp+store',med(t[r,:n,3]-t[r,:n,2]),'wait next S',med(np.r_[t[r,1:n,0]-t[r,:n-1,3],0]))
print('MMA: S0(j+1) issued - SL0(j)', med(t[0,:n,0]-t[1,:n,1]), ' PV0(j) issued - P0 arrive', med(t[0,:n,2]-t[1,:n,3]))
print('S0(j+1) issued -> softmax0 sees S(j+1)', med(t[1,1:n+1,0][:n-1]-t[0,:n-1,0]) if n>2 else '')
for j in range(20,23): print(j, t[0,j,:4], t[1,j,:4], t[2,j,:4])
