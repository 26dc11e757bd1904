import sys; sys.path.insert(0,'/root/repo')
import numpy as np, oracle
from synth import bank_corpus, init_rows
from paper_1905_09598_b200 import som
C = bank_corpus(5000, 3000, seed=5001); X = C.dense()
R = init_rows(X, 400, 3).astype(np.float64); W = (0.6*R + 0.4*X.mean(0, dtype=np.float64)).astype(np.float32)
m = som.SOM(20, 20, 3000, 1); m.set_weights(W)
som.som_set_map_precision(m.h, som.SOM_MAP_3XTF32); b1, b2, d1 = m.map(X)
som.som_set_map_precision(m.h, som.SOM_MAP_EXACT_F64); e1, e2, ed = m.map(X)
ob1, ob2, od1, m12, m23 = oracle.map_docs(W, X, want_margins=True)
assert np.array_equal(e1, ob1) and np.array_equal(ed, od1)
ab = np.abs(d1.astype(np.float64) - od1); rel = ab / od1
print("abs err: max %.3g p99 %.3g median %.3g" % (ab.max(), np.percentile(ab, 99), np.median(ab)))
print("rel err: max %.3g p99 %.3g median %.3g" % (rel.max(), np.percentile(rel, 99), np.median(rel)))
i = np.argmax(rel); print("worst doc D1 oracle", od1[i], "gpu", d1[i], "signed err", d1[i]-od1[i])
print("signed mean err", np.mean(d1.astype(np.float64) - od1), "D1 range", od1.min(), od1.max())
xn = (X.astype(np.float64)**2).sum(1); print("xnorm range", xn.min(), xn.max())
