"""Search level vectors whose plans cover the BLOCKED fused-group variants
(tests/test_parity_gpu.py BLOCKED_SHAPES).  Host-only: uses sgh_plan_describe."""
import itertools, re, sys
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
import paper_1309_0392_b200 as s, sgh_inputs as si
feats={}
cands=[]
for d in range(2,5):
    for lv in itertools.product(range(1,15),repeat=d):
        N=si.num_points(lv)
        if N>3_000_000 or N<1000: continue
        cands.append(lv)
import random; random.seed(1); random.shuffle(cands)
chosen=[]
for lv in cands[:6000]:
    for inv in (False,True):
        p=s.plan_describe(lv,inverse=inv)
        fs=set()
        for line in p.splitlines():
            m=re.search(r'FUSED W=(\d+) levels=\(([\d,]+)\) special=(-?\d+) bt=(-?\d+) aligned=(\d)',line)
            if not m or int(m.group(3))<0: continue
            W=int(m.group(1)); gl=[int(x) for x in m.group(2).split(',')]; j=int(m.group(3)); bt=int(m.group(4)); al=int(m.group(5))
            blocked = bt < gl[j]
            pos = 'first' if j==0 else ('last' if j==len(gl)-1 else 'mid')
            fs.add(('inv' if inv else 'hier', 'W1' if W==1 else 'Wcol', pos, 'blk%d'%(bt%3) if blocked else 'lat', al))
        new=fs-set(feats)
        if new:
            for f in new: feats[f]=lv
            chosen.append((lv,inv))
for f in sorted(feats): print(f, feats[f])
print(sorted(set(lv for lv,_ in chosen)), len(set(lv for lv,_ in chosen)))
