import sys; sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import numpy as np
from oracle.oracle import OCt, OracleContext
from paper_2104_03152_b200 import Context
from synthetic import CFG1, messages
from test_gpu_scheme import rand_ct

def diffinfo(o, a, b, lvl):
    for i in range(lvl+1):
        d = (a[i].astype(object) - b[i].astype(object)) % o.q[i]
        neq = np.count_nonzero(a[i] != b[i])
        dc = o.intt(i, np.array(d, dtype=np.uint64)).astype(object)
        q=o.q[i]; dcc = [int(x) - q if int(x) > q//2 else int(x) for x in dc]
        print(f"  limb {i}: {neq} words differ; coeff diff range {min(dcc)}..{max(dcc)}")

o = OracleContext(10, (50, 40, 40, 50, 50), 2, 9); g = Context(10, (50, 40, 40, 50, 50), 2, 9)
for lvl in (1, 2):
    x = rand_ct(o, lvl, 1, 10 + lvl)
    got = g.he_rescale(g.he_ct_import_words(x, lvl, 2.0**40)).words()[0]
    ref = o.rescale(OCt(x[0], lvl, 2.0**40)).words
    print("rescale lvl", lvl)
    for p in range(2): diffinfo(o, got[p], ref[p], lvl-1)

o = OracleContext(CFG1.logN, CFG1.bits, 1, 0); o.keygen([1])
g = Context(CFG1.logN, CFG1.bits, 1, 0); g.he_keygen([1])
lvl = 2
z = messages(1, 4096, seed=5)
pt = o.encode(z[0], 2.0**30, lvl)
ct = g.he_encrypt(g.he_pt_import_words(pt.words[None], lvl, 2.0**30), 100).words()[0]
ref = o.encrypt(pt, 100).words
print("encrypt cfg1")
for p in range(2): diffinfo(o, ct[p], ref[p], lvl)
