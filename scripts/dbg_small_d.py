import numpy as np, torch, sys
sys.path.insert(0, "/root/repo")
import paper_2603_00040_b200 as aq
from oracle import nvfp4_attn_oracle as orc
for (n_q,n_k,d,causal) in [(64,64,32,False),(64,64,16,False),(128,128,32,False),(64,64,48,False),(256,256,32,False)]:
    Q,K,V=orc.make_qkv(11+d,n_q,n_k,d)
    O,L,Op=orc.forward_training(Q,K,V,causal,n_q,n_k,32)
    cfg=aq.TileConfig(b_q=n_q,b_k=n_k,causal=causal)
    inst=[]
    outs=aq.flash_forward_training(Q,K,V,cfg,instrument=inst)
    tr=orc.oracle_forward(Q,K,V,causal=causal)
    pt=[r for r in inst if isinstance(r,aq.PTileRecord)][0].P_fq
    fl=np.sum(pt!=tr["P_fq"])
    err=np.linalg.norm(outs.O-O,axis=1)/np.linalg.norm(O,axis=1)
    print(n_q,d,"O",orc.rel_l2(outs.O,O),"Op",orc.rel_l2(outs.O_prime,Op),"L",np.abs(outs.L-L).max(),"flips",fl,"worst rows",np.argsort(err)[-3:],err.max())
    # compare device path too
    q,k,v=(torch.from_numpy(x).float().cuda() for x in (Q,K,V))
    o,lse,ohp,_=aq.attn_forward(q,k,v,train=True)
    print("   device O",orc.rel_l2(o.cpu().numpy(),O))
    # padded manually at 64 with d softmax
    if d<64:
        qp,kp,vp=(torch.nn.functional.pad(t,(0,64-d)) for t in (q,k,v))
        o2,_,_,_=aq.attn_forward(qp,kp,vp,train=True,softmax_scale=1/np.sqrt(d))
        print("   manual pad O",orc.rel_l2(o2[:, :d].cpu().numpy(),O), "Vf pad check", orc.rel_l2(aq.fake_quantize_cols(v).cpu().numpy(), tr["Vf"]))
