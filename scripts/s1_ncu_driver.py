"""ncu driver (tuning): a few segment + candidates calls on c2, for `ncu -k regex:stage1 ...`."""
import os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_2507_21433_b200.pipeline import MemSharePath
from synth import workloads
w = workloads.c2(seed=0)
b, sh = w.batch, w.shape
p = MemSharePath(b.tokens, b.seq_tok_off, b.gen_start, b.final, b.delim_ids, w.table, w.refcount, w.free_list,
                 w.free_count, None, None, 0, 0, w.num_blocks, sh.num_layers, sh.num_kv_heads, sh.num_kv_heads,
                 sh.head_dim, sh.block_size)
p.autosize(w.tau_s)
for _ in range(5):
    p.segment(); p.candidates(w.tau_s)
torch.cuda.synchronize()
