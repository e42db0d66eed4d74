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
