# how often the re-rank shortcut is attempted / passes its count check / decides the query (experiment build)
CHGPU_NVCC_EXTRA="-DCHGPU_SHORTCUT_STATS" python -m paper_1805_08995_b200.build --force > /dev/null 2>&1
CHGPU_NO_JOIN=1 python - <<'PY'
import numpy as np, paper_1805_08995_b200 as ch
m = ch.Matcher(0); fam = ch.build_hash_family(ch.FamilyParams()); m.set_family(fam)
import os
d = ch.make_dataset(64, 8192, seed=7, shape=os.environ.get("SHAPE", "uniform"))
ids = np.arange(64, dtype=np.uint32)
m.upload_many(ids, d); m.centering_reset(); m.centering_add_many(ids); m.centering_apply(); m.hash(ids)
pairs = ch.plan_exhaustive(64, 50, 4)
st = m.match_pairs_device(pairs, ch.MatchConfig())
q = st["query_points"]
print("RESULT rerank cases per query %.4f, count check passed %.4f of them, decided %.4f of them" % (st["verified_queries"] / q, st["distances"] / max(1, st["verified_queries"]), st["matches"] / max(1, st["verified_queries"])))
PY
python -m paper_1805_08995_b200.build --force > /dev/null 2>&1
