import sys, numpy as np
kb = np.load(sys.argv[1]); cta = int(sys.argv[2]) if len(sys.argv) > 2 else 0
e = kb[cta]; e = e[e[:,0]>0]; t0 = e[0,0]
for i,(a,b,c) in enumerate(e):
    print(i, round((a-t0)/1e3,2), round((b-a)/1e3,2), round((c-a)/1e3,2))
