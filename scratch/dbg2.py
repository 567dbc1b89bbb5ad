import sys; sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import numpy as np
from oracle.oracle import OCt, OracleContext
from paper_2104_03152_b200 import Context
from test_gpu_scheme import rand_ct
o = OracleContext(10, (50, 40, 40, 50, 50), 2, 9); g = Context(10, (50, 40, 40, 50, 50), 2, 9)
lvl = 2
x = rand_ct(o, lvl, 1, 12)
got = g.he_rescale(g.he_ct_import_words(x, lvl, 2.0**40)).words()[0]
np.save('gpurun_out/resc_x.npy', x); np.save('gpurun_out/resc_got.npy', got)
import torch
d = torch.from_numpy(x[0].copy().view(np.int64)).cuda()
g.he_ntt_inverse(d, 2, 3)
np.save('gpurun_out/resc_intt.npy', d.cpu().numpy().view(np.uint64))
