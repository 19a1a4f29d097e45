"""B200-native FV/RNS hot path of the CaRENets reference (arXiv 1901.10074).

Drop-in for the reference package ``hepack``'s lattice backend and CNN
layer API: the same names (SlotBackend contract, FvBackend, keygen,
layer_eval, infer, ...) with every homomorphic arithmetic step executed by
hand-written sm_100a CUDA kernels in ``_lib/libhefv.so`` (C-ABI:
include/hefv.h).  Importing the package needs no GPU; constructing an
FvBackend does, and fails loudly without the CUDA library.
"""

from .engine import Ciphertext, CostReport, SimBackend, SlotBackend, centered
from .errors import (
    CapacityError,
    DepthBudgetError,
    DimensionError,
    FormatError,
    HepackError,
    MemoryCapError,
    NativeError,
    ParamMismatchError,
    RangeCertificateError,
)
from .params import BackendParams, load_profiles, profile, profile_names

__version__ = "0.1.0"


def __getattr__(name):
    # GPU-backed modules load lazily so that `import paper_1901_10074_b200`
    # works on hosts without torch/CUDA (host-only tests, tooling).
    if name in ("FvBackend", "FvParams", "KeySet", "SwitchKey", "FvCiphertext", "keygen",
                "run_sequence", "fv_conformance", "FvContext"):
        from . import fv

        return getattr(fv, name)
    if name in ("ConvSpec", "FcSpec", "NetworkSpec", "PackedVector", "SquareSpec", "WeightRow",
                "compile_conv", "compile_fc", "decrypt_logits", "infer", "layer_eval",
                "pack_image", "square_activation"):
        from . import inference

        return getattr(inference, name)
    raise AttributeError(name)
