import sys; sys.path.insert(0,'.')
import paper_2601_05524_b200 as dbl
cfg=dbl.transformer_config("tiny-qwen", seed=21, max_seq=2048)
tgt=dbl.Transformer(cfg)
prompt=list(range(1,30))
ar=dbl.run_vanilla_ar(tgt,prompt,900)
print("AR stream tail", ar.output[:60], len(set(ar.output)))
stream=prompt+ar.output
prior=[stream[i:i+64] for i in range(0,len(stream)-64,8)]
for g in (24, 40, 64):
  st=dbl.HierarchicalDatastore(3,10); dbl.build_prior(st,prior,len(prior))
  r=dbl.run(tgt,tgt,st,prompt,900,dbl.PipelineOptions(gamma=g,depth=10))
  print(g, r.output==ar.output, max(t["pending"] for t in r.traces), [ (t["pending"],t["draft_len"],t["kind"],t["target_matched"]) for t in r.traces[:12]])
  print(r.traces[3])
