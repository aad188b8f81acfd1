import sys, numpy as np
sys.path.insert(0, '.')
from paper_2510_22506_b200 import _native
def unf(x,k):
    rest=[m for m in range(x.ndim) if m!=k]; return np.transpose(x,[k]+rest).reshape((x.shape[k],-1),order='F')
rng=np.random.default_rng(0)
for dims,k,S in [((256,64,8),2,64),((256,64,8),1,64),((256,64,8),0,64),((128,32,1),1,64)]:
    x=np.asfortranarray(rng.standard_normal(dims).astype(np.float32)); p=int(np.prod(dims))//dims[k]
    m=np.asfortranarray(rng.standard_normal((p,S)).astype(np.float32))
    ref=unf(x.astype(np.float64),k)@m.astype(np.float64)
    y=_native.selftest_stream(x,m,k,True); ys=_native.selftest_stream(x,m,k,False)
    print(dims,k,S,'tc err',np.linalg.norm(y-ref)/np.linalg.norm(ref),'simt err',np.linalg.norm(ys-ref)/np.linalg.norm(ref))
    print('  ref[:3,:3]',ref[:3,:3].ravel()); print('  tc [:3,:3]',y[:3,:3].ravel())
    # diagnostics: is it transposed / scaled
    nz=np.count_nonzero(y); print('  nonzero',nz,'of',y.size, 'max',np.abs(y).max(), 'refmax',np.abs(ref).max())
# unit test: x = ones-pattern to decode layout
dims=(128,32,1); k=1; S=64
x=np.zeros(dims,np.float32,order='F'); x[0,0,0]=1.0  # X_(1)[i=0, p=0]
m=np.zeros((128,S),np.float32,order='F'); m[0,:]=np.arange(S)
y=_native.selftest_stream(x,m,k,True); print('delta test: y[0,:8]',y[0,:8],'nnz',np.count_nonzero(y), np.argwhere(y!=0)[:10].tolist())
