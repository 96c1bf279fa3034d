import json, numpy as np, sys
d=json.load(open('gpurun_out/mega_trace.json'))
tasks=np.array(d['tasks']); tr=np.array(d['trace'],dtype=np.int64)
types=tasks[:,0]&0xff; ops=tasks[:,0]>>8
# epi units of op 15: look at timings
o=int(sys.argv[1]) if len(sys.argv)>1 else 15
idx=np.where((types==1)&(ops==o))[0]
print(idx[:10], tr[idx[:10],0]/1e3, tr[idx[:10],1]/1e3)
