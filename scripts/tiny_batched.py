import torch, sys
sys.path.insert(0, '/root/repo')
import paper_1309_0392_b200 as sgh, sgh_inputs as si
b = sgh.GridBatch(si.combination_set(4, 12))
b.fill_uniform(si.SEED)
b.hierarchize()
torch.cuda.synchronize()
print("ok", sgh.launch_count())
