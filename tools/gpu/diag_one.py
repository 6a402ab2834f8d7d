
import sys, numpy as np, torch
sys.path.insert(0, ".")
import oracle, paper_2602_21600_b200 as aqr
from tests._cases import case
name,layout,tr,vb=sys.argv[1],sys.argv[2],sys.argv[3],int(sys.argv[4])
c=case(name); x=torch.from_numpy(c.w.x).cuda()
codes,quant=aqr.encode(x,sample_idx=torch.from_numpy(c.sample).cuda(),p_max=5.0,delta_override=c.delta_override)
ix=aqr.upload_index(codes,x,quant,c.graph,metric=c.w.metric,layout=layout)
q=torch.from_numpy(np.ascontiguousarray(c.w.q[:8])).cuda(); k=c.w.k
p=dict(k=k,**oracle.ef_mapping(48,k))
ids,d,t=aqr.search(ix,q,trace=True,visited_bits=vb,traversal=tr,**p); torch.cuda.synchronize()
ids,d=aqr.search(ix,q,visited_bits=vb,traversal=tr,**p); torch.cuda.synchronize()
print("OK")
