"""Drop-in binding of the GPU backend into the reference's own modules.

The reference's callers (``hepack.inference``, ``hepack.matrix``,
``hepack.fv.run_sequence`` / ``fv_conformance``, ``hepack.serialize``) only
use the ``SlotBackend`` contract (engine.py:124-350), which ``FvBackend``
implements name for name, so they run unchanged on it.  Two places in the
reference need more than duck typing, and this module supplies both without
ever importing the reference (the caller passes its modules in):

* ``serialize.read_ciphertext`` accepts an FV record only when
  ``isinstance(backend, hepack.fv.FvBackend)`` (serialize.py:108-110).
  ``gpu_backend_class(hepack_fv)`` returns ``GpuFvBackend``, a subclass of
  both this package's ``FvBackend`` and the caller's ``FvBackend``
  (SURVEY.md 8b): every method resolves to the GPU implementation first, the
  reference's ``__init__`` never runs (no CPU keygen), and the reference's
  host ``FvCiphertext`` records it reads are validated and uploaded by
  ``FvBackend.dev``.
* ``inference.layer_eval`` (inference.py:261-349) evaluates one row at a
  time.  Its result is identical on this backend (tests/test_dropin.py), but
  the batched planner is ~10^3x faster, so the reference gains a three-line
  dispatch at the top of ``layer_eval`` that calls
  ``backend.layer_eval_batched`` when the backend has one.
  ``layer_eval_hook(original)`` is exactly that dispatch, as a wrapper.
"""

from __future__ import annotations

from .fv import FvBackend

_CLASSES: dict = {}


def gpu_backend_class(hepack_fv):
    """``class GpuFvBackend(FvBackend, hepack_fv.FvBackend)``, cached per module."""
    base = hepack_fv.FvBackend
    cls = _CLASSES.get(base)
    if cls is None:
        cls = type("GpuFvBackend", (FvBackend, base), {
            "__doc__": "GPU FvBackend that is also an instance of the caller's FvBackend.",
            "__module__": __name__,
        })
        _CLASSES[base] = cls
    return cls


def layer_eval_hook(original):
    """The dispatch the reference's ``layer_eval`` gains:
    backends exposing ``layer_eval_batched`` evaluate the whole layer in
    batched launches; every other backend runs ``original`` unchanged."""

    def layer_eval(backend, rows, x, skip_zero_segments=True, threads=1, scale_factor=1):
        batched = getattr(backend, "layer_eval_batched", None)
        if batched is not None:
            return batched(rows, x, skip_zero_segments, scale_factor)
        return original(backend, rows, x, skip_zero_segments=skip_zero_segments,
                        threads=threads, scale_factor=scale_factor)

    layer_eval.__wrapped__ = original
    layer_eval.__doc__ = original.__doc__
    return layer_eval
