"""Images queued on two CUDA streams (the config-5 image-stream schedule of
bench.py) produce exactly the ciphertexts of the one-stream run: every piece
of per-call device state -- key-switch workspaces (per stream), pinned plan
staging (a pool reused only after its copy completed), stream-ordered
temporaries -- is safe under concurrency.  Small aux-basis parameters
(N = 1024, k = 10) so both key-switch paths' shared state is exercised."""

import numpy as np
import pytest

from oracle.fv_oracle import limb_digest
from paper_1901_10074_b200 import inference as I
from paper_1901_10074_b200.configs import config_network
from paper_1901_10074_b200.params import BackendParams

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("bits", [120, 300], ids=["per_prime_ks", "aux_ks"])
def test_two_streams_equal_one_stream(bits):
    import torch

    from paper_1901_10074_b200.fv import FvBackend

    p = BackendParams(ring_dimension=1024, coeff_modulus_bits=bits, plain_modulus=12289,
                      slot_count=512, depth_budget=6)
    _, net = config_network(1)
    rng = np.random.default_rng(4)
    imgs = [rng.integers(0, 8, (1, 16, 16), dtype=np.int64) for _ in range(4)]

    def run(streams):
        be = FvBackend(p, rng=np.random.default_rng(21))
        outs = []
        for i, img in enumerate(imgs):
            ctx_stream = torch.cuda.stream(streams[i % len(streams)]) if streams else None
            if ctx_stream is None:
                outs.append(I.infer(be, net, I.pack_image(be, img)))
            else:
                with ctx_stream:
                    outs.append(I.infer(be, net, I.pack_image(be, img)))
        torch.cuda.synchronize()
        return be, outs

    be1, seq = run(None)
    s = [torch.cuda.Stream(), torch.cuda.Stream()]
    be2, par = run(s)
    for a, b in zip(seq, par):
        assert [limb_digest(ct.parts) for ct in a.cts] == [limb_digest(ct.parts) for ct in b.cts]
    for a, b in zip(seq, par):
        assert list(I.decrypt_logits(be1, a)) == list(I.decrypt_logits(be2, b))
