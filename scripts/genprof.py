import sys
sys.path.insert(0, '.')
import numpy as np
import paper_1805_08995_b200 as ch
m = ch.Matcher(0)
fam = ch.build_hash_family(ch.FamilyParams())
m.set_family(fam)
data = ch.make_dataset(32, 8192, seed=7)
m.centering_reset()
for i in range(32):
    m.upload(i, data[i]); m.centering_add(i)
m.centering_apply(); m.hash(np.arange(32, dtype=np.uint32))
pairs = ch.plan_exhaustive(32, 8, 2)
print(m.match_pairs_device(pairs, ch.MatchConfig(top_k=33)))
