import sys; sys.path.insert(0,'.')
import numpy as np, torch
from paper_1901_10074_b200.configs import config_params
from paper_1901_10074_b200.fv import FvBackend, FvCiphertext
from oracle import fv_oracle as O
name = sys.argv[1] if len(sys.argv) > 1 else "retina"
from paper_1901_10074_b200.params import profile
p = profile(name)
be = FvBackend(p, rng=np.random.default_rng(1))
octx = O.OracleContext(O.OracleParams.from_backend(p))
rng = np.random.default_rng(3)
parts = [np.stack([rng.integers(0, q, p.ring_dimension) for q in octx.fp.q_primes]) for _ in range(2)]
vec = rng.integers(0, 9, p.slot_count)
ob = O.make_backend_class()
# oracle cmult without keys: replicate _cmult
class Dummy: pass
m = None
t = octx.t
ev = np.zeros(octx.n, dtype=octx.t_ntt.dtype); ev[octx.slot_to_ev] = np.asarray(vec, dtype=octx.t_ntt.dtype) % t
poly = octx.t_ntt.inv(ev)
mm = np.asarray(poly) % t; mm = np.where(mm > t//2, mm - t, mm)
want = []
for c in parts:
    out = np.empty_like(c)
    for j, tr in enumerate(octx.q_ntt):
        out[j] = tr.inv(tr.fwd(c[j]) * tr.fwd(mm % tr.p) % tr.p)
    want.append(out)
got = be.cmult(FvCiphertext(parts, 0, p), vec).parts
print("cmult equal", all(np.array_equal(a, b) for a, b in zip(got, want)))
# NTT of ct vs oracle natural
ctx = be.ctx
dev = torch.from_numpy(np.stack(parts).astype(np.int32)).cuda()
nat_fwd = ctx.ntt_q(dev.view(-1, ctx.k, ctx.n), natural=True).cpu().numpy().reshape(2, ctx.k, ctx.n)
print("ntt natural equal", all(np.array_equal(nat_fwd[0][j], octx.q_ntt[j].fwd(parts[0][j])) for j in range(ctx.k)))
# encode
gp = be.encode(vec)
print("encode equal", np.array_equal(np.asarray(gp, dtype=object), np.asarray(poly, dtype=object)))
# plaintext NTT in device order (Montgomery form) vs oracle
mdev = be._cmult_plain_dev(np.asarray(be.as_plain(vec))[None])[0].cpu().numpy().astype(np.int64)
brev = ctx.brev
ok = True
for j, tr in enumerate(octx.q_ntt):
    ref = tr.fwd(mm % tr.p)           # natural order
    mine = np.empty_like(ref); mine[brev] = mdev[j]  # device -> natural
    rinv = pow(1 << 32, -1, tr.p)
    mine = (mine.astype(object) * rinv % tr.p).astype(np.int64)
    if not np.array_equal(mine, ref): ok = False; print("plain ntt mismatch at prime", j); break
print("plain ntt (montgomery) equal", ok)
# mul_plain with the correct m_ntt vs oracle
out = torch.empty_like(dev)
mt = torch.from_numpy(mdev.astype(np.int32)).cuda()
ctx.call("hefv_mul_plain", dev.data_ptr(), mt.data_ptr(), out.data_ptr(), 1, 2, 1, ctx.stream())
o = out.cpu().numpy().astype(np.int64)
print("mul_plain equal", all(np.array_equal(o[i], want[i]) for i in range(2)))
# (a) mul_plain with m = 1 (Montgomery form R mod p) must return the input
R = np.array([[(1 << 32) % q] * ctx.n for q in octx.fp.q_primes], dtype=np.int64)
mt1 = torch.from_numpy(R.astype(np.int32)).cuda()
ctx.call("hefv_mul_plain", dev.data_ptr(), mt1.data_ptr(), out.data_ptr(), 1, 2, 1, ctx.stream())
o = out.cpu().numpy().astype(np.int64)
print("mul_plain identity", all(np.array_equal(o[i], parts[i]) for i in range(2)))
# (b) standalone fwd (device order) then inverse (device order) roundtrip
f = ctx.ntt_q(dev.view(-1, ctx.k, ctx.n))
b = ctx.ntt_q(f, inverse=True).cpu().numpy().astype(np.int64).reshape(2, ctx.k, ctx.n)
print("ntt dev-order roundtrip", all(np.array_equal(b[i], parts[i]) for i in range(2)))
# (c) device-order fwd vs natural fwd (permuted)
fd = f.cpu().numpy().astype(np.int64).reshape(2, ctx.k, ctx.n)
print("dev order == bitrev(natural)", np.array_equal(fd[0][0][brev], nat_fwd[0][0]) or np.array_equal(fd[0][0], nat_fwd[0][0][brev]))
