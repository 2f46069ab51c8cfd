import sys; sys.path.insert(0,'.')
import numpy as np, torch
import paper_2605_29346_b200 as gb
from paper_2605_29346_b200.models import GCNTrainer
MB=2**20
def m(tag): torch.cuda.synchronize(); print(f"{tag:40s} alloc {torch.cuda.memory_allocated()/MB:9.1f} MB  peak {torch.cuda.max_memory_allocated()/MB:9.1f} MB", flush=True)
V,E=232965,114615892
g=gb.generate(gb.GraphGenSpec("power-law",V,E,exponent=2.1),42); m("generate")
g.csc(); m("csc")
_=g.targets; m("host targets")
g.csr_coalesced(); m("csr_coalesced")
g.csc_coalesced(); m("csc_coalesced")
g.drop_csc(); g.release_device_targets(); torch.cuda.empty_cache(); m("released canonical")
torch.cuda.reset_peak_memory_stats(); m("reset")
tr=GCNTrainer(g,602,16,41,seed=42,coalesced=True); m("trainer init")
X=torch.rand(V,602).pin_memory(); y=torch.randint(0,41,(V,)).pin_memory()
tr.set_inputs(X,y); m("set inputs")
tr.step(); m("step")
tr.capture(); m("capture")
tr.run(); m("run")
print("plans", {k: [ (kk, buf.numel()*4/MB) for kk,(p,buf) in op._plans.items()] for k,op in (("A",tr.A),("AT",tr.AT))})
print("graph device bytes", g.device_nbytes()/MB)
