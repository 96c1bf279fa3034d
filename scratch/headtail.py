import json, sys, numpy as np
d = json.load(open(sys.argv[1])); tasks = np.array(d["tasks"]); tr = np.array(d["trace"], dtype=np.int64)
kb = np.load(sys.argv[2])
types = tasks[:, 0] & 0xff; ops = tasks[:, 0] >> 8
entry = kb[:, 1023, 0]; exitt = kb[:, 1023, 1]
valid = entry > 0
t0 = entry[valid].min()
print("kernel entry spread (us): first 0, last %.2f" % ((entry[valid].max() - t0) / 1e3))
pre = tr[types == 2]; fin = tr[types == 3]
pre = pre[pre[:, 4] > 0]; fin = fin[fin[:, 4] > 0]
print("prep: start %.2f .. end %.2f" % ((pre[:, 0].min() - t0) / 1e3, (pre[:, 4].max() - t0) / 1e3))
g = types == 0
r = tr[g]
print("op0 Bdep %.2f" % ((r[ops[g] == 0][:, 0].min() - t0) / 1e3))
last_op = ops[g].max()
print("last op done %.2f" % ((r[ops[g] == last_op][:, 4].max() - t0) / 1e3))
print("final: spin-done %.2f .. end %.2f" % ((fin[:, 0].min() - t0) / 1e3, (fin[:, 4].max() - t0) / 1e3))
print("kernel exit: first %.2f last %.2f" % ((exitt[valid].min() - t0) / 1e3, (exitt[valid].max() - t0) / 1e3))
