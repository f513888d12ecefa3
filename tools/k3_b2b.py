import sys, torch
sys.path.insert(0, '.')
import bench
from paper_2010_02164_b200 import DecodeConfig, Vocabulary
from paper_2010_02164_b200 import _native as N
from paper_2010_02164_b200.engine import SearchEngine
from paper_2010_02164_b200.scorers import DeviceHashScorer
w = dict(bench.WORKLOADS["wmt19_k50"], N=300)
corpus = bench._corpus(w)
vocab = Vocabulary(w["V"], 0, 2)
cfg = DecodeConfig(k=50, n=128, epsilon=1/6, delta=1.5, max_candidates=5, max_len=256)
eng = SearchEngine(cfg, vocab)
sc = DeviceHashScorer(vocab, 7, scale=0.5, power=0, eos_bias=7.5, dtype="bf16")
# run a few steps of the sync driver to get a populated state, then stop
eng.load_corpus(corpus); sc.bind(eng)
eng.schedule(first=True, remove=False, admit=N.VS_ADMIT_VARSTREAM, select=N.VS_SELECT_MIN_LT)
st = eng.read_status()
for _ in range(5):
    eng._step(sc, st, phase="stream", admit=N.VS_ADMIT_VARSTREAM, select=N.VS_SELECT_MIN_LT)
    st = eng.read_status()
print("live", st[N.ST_NLIVE], "R", st[N.ST_R])
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(30)]
for e0, e1 in ev:
    e0.record(); eng.schedule(first=False, remove=False, admit=N.VS_ADMIT_NONE, select=N.VS_SELECT_MIN_LT); e1.record()
torch.cuda.synchronize()
print("K3 standalone b2b us:", sorted(round(a.elapsed_time(b)*1e3,1) for a,b in ev))
# interleave with a big kernel that thrashes the icache (K1 full width)
x = torch.randn(2000, 42024, device="cuda").to(torch.bfloat16)
from paper_2010_02164_b200.search import row_lse_topm
ts=[]
for i in range(20):
    row_lse_topm(x, 5)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); eng.schedule(first=False, remove=False, admit=N.VS_ADMIT_NONE, select=N.VS_SELECT_MIN_LT); e1.record()
    torch.cuda.synchronize(); ts.append(round(e0.elapsed_time(e1)*1e3,1))
print("K3 after K1 us:", sorted(ts))
# 20 back-to-back K3 launches inside one CUDA graph: no host gaps, warm instruction cache
g = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    eng._sp = None
    with torch.cuda.graph(g):
        for _ in range(20):
            eng.schedule(first=False, remove=False, admit=N.VS_ADMIT_NONE, select=N.VS_SELECT_MIN_LT)
torch.cuda.current_stream().wait_stream(s)
g.replay(); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
print("K3 in-graph b2b us per launch:", round(e0.elapsed_time(e1) * 1e3 / 20, 2))
