import sys; sys.path.insert(0,'.')
import json
import numpy as np, torch
from paper_1901_10074_b200 import inference as I, _native as nat
from paper_1901_10074_b200.configs import config_network, config_params
from paper_1901_10074_b200.fv import FvBackend
from oracle.fv_oracle import limb_digest
g=json.load(open('tests/golden/retina.json'))
img, net = config_network(2)
be = FvBackend(config_params(2), rng=np.random.default_rng(1234))
pv = I.pack_image(be, img)
rows = I.compile_conv(net.layers[0], pv.slots_used)
ctx=be.ctx; n=ctx.n; t=be.params.plain_modulus
r=rows[0]
vec=r.segment_dense(0, be.params.slot_count)
# dense encode
pd = be._encode_dev(be.as_plain(vec)[None])
# sparse encode
sel = r.positions//8192==0
d_ptr=nat.to_device(np.array([0,int(sel.sum())],dtype=np.int32))
d_idx=nat.to_device((r.positions[sel]%8192).astype(np.int32))
d_val=nat.to_device(np.mod(r.values[sel].astype(np.int64),t).astype(np.uint64).view(np.int64))
ps=torch.empty((1,n),dtype=torch.int64,device='cuda')
ctx.call("hefv_encode_sparse", d_ptr.data_ptr(), d_idx.data_ptr(), d_val.data_ptr(), ps.data_ptr(), 1, ctx.stream())
print("encode dense==sparse", torch.equal(pd, ps))
m1=be._rns_plain(pd,1,True,False); m2=be._rns_plain(ps,1,True,False)
print("plain_to_rns equal", torch.equal(m1,m2))
# cmult via mul_plain vs rows_mac
a=be.cmult(pv.cts[0], vec)
xin=torch.stack([pv.cts[0].device()[:2]]).contiguous()
x_ntt=ctx.to_mont(ctx.ntt_q(xin.view(-1,ctx.k,n)).view_as(xin))
acc=torch.empty((1,2,ctx.k,n),dtype=torch.int32,device='cuda')
rp=nat.to_device(np.array([0,1],dtype=np.int32)); sg=nat.to_device(np.array([0],dtype=np.int32))
ctx.call("hefv_rows_mac", x_ntt.data_ptr(), m2.data_ptr(), rp.data_ptr(), sg.data_ptr(), acc.data_ptr(), 1, ctx.stream())
print("rows_mac == cmult", torch.equal(acc[0], a.device()))
sub=[rows[i] for i in g["rows_pick"]]
pa = I.layer_eval(be, sub, pv)
sb = I._serial_layer_eval(be, sub, pv, True, 1)
print("planner golden", limb_digest(pa.cts[0].parts)==g["rows_out"][0], "serial golden", limb_digest(sb.cts[0].parts)==g["rows_out"][0])
