import sys, os, torch
sys.path.insert(0, os.getcwd())
import paper_2110_01899_b200 as rf, synthetic
cfg = synthetic.CONFIGS[3]
X = torch.from_numpy(synthetic.make_X(cfg)).to(torch.bfloat16).cuda()
W = torch.from_numpy(synthetic.make_W(cfg))[:8192].to(torch.bfloat16).cuda()
ctx = rf.Context(0); ctx.set_option("k4_cl8", 1); ctx.set_option("verbose", 1)
rf.rf_gram(X, W, act=cfg.act, ctx=ctx); torch.cuda.synchronize(); print("done")
