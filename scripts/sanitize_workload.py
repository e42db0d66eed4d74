import sys; sys.path[:0]=[".", "tests", "oracle"]
import numpy as np, torch
from paper_2601_13345_b200 import corpus, synth, native, engine
import test_corpus_parity as T
rt = native.get_runtime(0)
text, offs = synth.ptx_corpus(seed=21, n_kernels=40, lo=20, hi=800)
zoo = ".visible .entry zoo()\n{\nL0:\n" + "\n".join("\t" + st for st in T.OPERAND_ZOO) + "\n\tret;\n}\n"
from edge_cases import EDGE_CASES
blobs = [text[offs[i]:offs[i+1]] for i in range(40)] + [zoo.encode()] + [v.encode() for v in EDGE_CASES.values()]
corp = corpus.upload_corpus(b"".join(blobs), np.cumsum([0]+[len(b) for b in blobs]))
lex, fl = corpus.analyze_corpus(corp)
h = corpus.lex_histogram(corp)
l1 = corpus.lex_records_single_pass(corp)
f1 = corpus.kernel_features(corp, l1)
e, t = synth.candidate_cloud(seed=5, n=4*3248, kind="tied")
occ = (np.random.default_rng(1).integers(1, 6, e.size) / 5.0)
d = lambda x: rt.to_device(torch.from_numpy(np.ascontiguousarray(x)))
engine.skyline_groups(d(e), d(t), 4, 3248, rho=0.95)
engine.skyline_groups(d(e), d(t), 4, 3248, rho=0.95, occ=d(occ), tie=d(np.random.default_rng(2).permutation(3248).astype(np.int32)))
engine.skyline(d(e), d(t), rho=0.0, cap_front=4096, occ=d(occ))
torch.cuda.synchronize()
print("sanitizer workload done", int((fl.status.cpu()!=0).sum()))
# ---- round 2: fused explore, factored grid kernel, streaming pre-filter (2 and 3 objectives), sort-based finish ----
import os
from paper_2601_13345_b200 import specs
os.environ["FFB_SKYLINE_PREFILTER_MIN"] = "1000"
a, p = specs.default_architecture(), specs.default_calibration()
sp = engine.spec_rows([(a, p, 65536)])
shp = engine.shape_rows([tuple(x) for x in engine.enumerate_shapes(sp[0], 0, list(range(1, 257)))])
feat, res = synth.feature_rows(seed=5, n_kernels=6)
caps = np.array([100.0, 150.0, 200.0, 250.0])
df, dr = engine.features_tensor(feat), engine.resources_tensor(res)
engine.score_grid(df, dr, sp, shp, caps, want=("t", "e"), check=False)
engine.explore_groups(df, dr, sp, shp, caps, rho=0.95)
e2, t2 = synth.candidate_cloud(seed=6, n=60_000, kind="uniform")
engine.skyline(d(e2), d(t2), rho=0.9, cap_front=4096)
engine.skyline(d(e2), d(t2), rho=0.0, cap_front=4096, occ=d(np.random.default_rng(3).integers(1, 9, e2.size) / 8.0))
e3, t3 = synth.candidate_cloud(seed=7, n=60_000, kind="tied")
engine.skyline(d(e3), d(t3), rho=0.0, cap_front=60_000)
torch.cuda.synchronize()
print("round-2 sanitizer workload done")
