import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
import paper_1708_09495_b200 as bsg
n = int(sys.argv[1]); p = int(sys.argv[2]); G = int(sys.argv[3])
keys = bsg.generate_uniform_keys_device(n, 3).view(torch.int32)
grp = bsg._lib.GroupContext([0] * G)
rng = [bsg.radix.group_range(n, p, G, g) for g in range(G)]
blocks = [keys[o:o + s].clone() for o, s in rng]
bsg.radix.group_sort_blocks(grp, blocks, n, p, 256, rounds=(None if len(sys.argv) < 5 else int(sys.argv[4])))
torch.cuda.synchronize()
print("ok", n, p, G)
