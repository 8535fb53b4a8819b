import numpy as np, sys
a=np.load(sys.argv[1]); b=np.load(sys.argv[2])
for k in a.files:
    x,y=a[k],b[k]
    print(k, 'bitwise equal' if np.array_equal(x,y) else f'DIFF max {np.abs(x-y).max()} count {(x!=y).sum()} first_iter {np.argwhere(x!=y)[0] if (x!=y).any() else None}')
