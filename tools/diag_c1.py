import sys, os, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import train_ref
from paper_2502_19913_b200.configs import get_config
from paper_2502_19913_b200.executor import Trainer
from paper_2502_19913_b200.model import init_params, synthetic_tokens
rc = get_config("C1"); sch = rc.schedule()
params = init_params(rc.model, rc.layers, seed=0)
tokens = synthetic_tokens(rc.model, rc.M, rc.b, rc.T, seed=1234)
agents = sorted(a.id for a in sch.agents)
mbs = train_ref.mb_stage_sequences({a: sch.paths[a].stages for a in agents}, agents, rc.M)
ref = train_ref.iteration(rc.model, rc.layers, params, mbs, tokens, update=False)
for graphs in (False, True):
    tr = Trainer(sch, rc.topology(), rc.sim_config(), rc.model, rc.assignment, b=rc.b, T=rc.T, split=rc.split, params=params, use_graphs=graphs)
    r = tr.step(tokens)
    print("graphs", graphs, "loss", r["loss"], "ref", ref["loss"])
    print(" mb", [round(x, 4) for x in tr.mb_loss.tolist()])
    print(" rf", [round(x, 4) for x in ref["mb_loss"]])
    g = tr.grads(); g = [g[st] for st in range(4)]
    for st in range(4):
        a = torch.cat([g[st][k].reshape(-1) for k in sorted(g[st])]); b = torch.cat([ref["grads"][st][k].reshape(-1) for k in sorted(ref["grads"][st])])
        print(" stage", st, "cos", torch.nn.functional.cosine_similarity(a.double(), b.double(), dim=0).item(), "ratio", (a.norm()/b.norm()).item())
        for k in sorted(g[st])[:6]:
            print("   ", k, (g[st][k].norm()/ref['grads'][st][k].norm()).item())
print("ops", [(o.kind, o.node, o.mb, o.slot, o.pos) for o in tr.ops][:30])
