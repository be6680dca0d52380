"""Reference-side binding: the reference package's own entry points, run on the B200.

This is the module INTEGRATION.md section 2 describes as ``pkg/src/batchrand/_b200.py``,
shipped here so that it is executed and tested (tests/test_refbind.py).  ``bind(ref)`` takes
the imported reference package (``batchrand``, e.g. from ``baseline/_ref`` -- see
tools/vendor_reference.sh) and returns device-backed versions of its hot-path functions that
take the reference's OWN objects and raise the reference's OWN exception classes:

=============================================  ===================================================
reference (pkg/src/batchrand/...)              device call (include/batchrand_b200.h)
=============================================  ===================================================
shuffle.py:149 ``shuffle_batched``             br_shuffle_stream
shuffle.py:80  ``shuffle_unbatched``           br_shuffle_stream(unbatched=1)
shuffle.py:137 ``partial_shuffle_batch``       br_shuffle_stream_segments
shuffle.py:228 ``shuffle_naive_batched``       br_shuffle_naive_stream
batched.py:102 ``roll_batch``                  br_roll_batches (+ br_roll_check), br_roll_batch64
batched.py:85  ``roll_batch_known_threshold``  br_roll_batches
batched.py:126 ``roll_batch_naive``            br_roll_batches_naive
batched.py:69  ``digit_pass``                  br_digit_pass / br_roll_batch64
=============================================  ===================================================

Sources: the reference's ``Pcg64Source`` (wordsource.py:70-89), ``LehmerSource`` (:51-67),
``ChaChaSource`` (:136-164) and 64-bit ``FixedSequenceSource`` (:191-207) are read through
their attributes and advanced by exactly the words the device consumed.  Schedules
(shuffle.py:22-49), ``BatchSpec`` (batched.py:26-51) and ``RadixBases`` (mixed_radix.py:18-37)
are the reference's objects.

``install(ref)`` patches the reference package in place (module attributes and the
``cli.ALGORITHMS`` registry, cli.py:44-49) and returns an ``uninstall`` callable;
``register_algorithms(ref.cli)`` only adds the ``*_b200`` rows to the CLI registry so that
``batchrand bench`` times the GPU next to the CPU algorithms.

There is no CPU fallback here either: without a CUDA device every call raises.
"""

from __future__ import annotations

import functools
import types

from . import batchrand as B
from . import errors as E

_ERR_NAMES = ("SourceExhausted", "BoundOverflow", "DigitOutOfRange", "ValueOutOfRange", "UnknownGenerator",
              "UnknownAlgorithm", "NoCrossover", "InsufficientTrials")


def _translate(ref):
    """Decorator mapping this package's exceptions onto the reference's classes of the same
    name (errors.py:4-37), so reference callers' ``except`` clauses keep working."""
    ref_errors = getattr(ref, "errors", ref)
    table = []
    for name in _ERR_NAMES:
        ours, theirs = getattr(E, name, None), getattr(ref_errors, name, None)
        if ours is not None and theirs is not None:
            table.append((ours, theirs))

    def deco(fn):
        @functools.wraps(fn)
        def wrapper(*a, **kw):
            try:
                return fn(*a, **kw)
            except E.BatchRandError as exc:
                for ours, theirs in table:
                    if isinstance(exc, ours):
                        raise theirs(str(exc)) from exc
                raise

        return wrapper

    return deco


def _schedule(s):
    """The reference's ShuffleSchedule (entries, max_batch, word_bits) as this package's."""
    if isinstance(s, B.ShuffleSchedule):
        return s
    return B.ShuffleSchedule(entries=tuple((int(m), int(k)) for m, k in s.entries), max_batch=int(s.max_batch),
                             word_bits=int(s.word_bits))


def _bases(rb):
    return B.RadixBases.of(tuple(int(b) for b in rb.bases), int(rb.bits))


def bind(ref) -> types.SimpleNamespace:
    """Device-backed hot-path functions over the reference package ``ref``'s objects."""
    tr = _translate(ref)
    BatchResult = ref.BatchResult
    default = ref.DEFAULT_SCHEDULE

    @tr
    def shuffle_batched(source, z, schedule=default, check_bounds=False):
        """shuffle.py:149-225."""
        return B.shuffle_batched(source, z, _schedule(schedule), check_bounds)

    @tr
    def shuffle_unbatched(source, z):
        """shuffle.py:80-97."""
        return B.shuffle_unbatched(source, z)

    @tr
    def shuffle_naive_batched(source, z):
        """shuffle.py:228-266."""
        return B.shuffle_naive_batched(source, z)

    @tr
    def partial_shuffle_batch(source, z, n, k, u):
        """shuffle.py:137-146."""
        return B.partial_shuffle_batch(source, z, n, k, u)

    def _spec(spec, keep_threshold):
        t = spec.precomputed_threshold if keep_threshold else None
        return B.BatchSpec(_bases(spec.bases), precomputed_threshold=t, upper_bound=spec.upper_bound)

    @tr
    def roll_batch(source, spec):
        """batched.py:102-123."""
        r = B.roll_batch(source, _spec(spec, False))
        return BatchResult(tuple(r.digits), r.words_consumed, r.threshold_computed, r.final_remainder)

    @tr
    def roll_batch_known_threshold(source, spec):
        """batched.py:85-99."""
        if spec.precomputed_threshold is None:
            raise ValueError("spec has no precomputed threshold")
        r = B.roll_batch_known_threshold(source, _spec(spec, True))
        return BatchResult(tuple(r.digits), r.words_consumed, r.threshold_computed, r.final_remainder)

    @tr
    def roll_batch_naive(source, bases):
        """batched.py:126-128."""
        return tuple(B.roll_batch_naive(source, _bases(bases)))

    @tr
    def digit_pass(r0, bases):
        """batched.py:69-82."""
        d, rk = B.digit_pass(r0, _bases(bases))
        return tuple(d), rk

    def _shuffle_2(source, z):
        return shuffle_batched(source, z, ref.default_schedule(2))

    def _shuffle_6(source, z):
        return shuffle_batched(source, z, ref.default_schedule(6))

    # cli.py:44-49 names with a _b200 suffix
    algorithms = {
        "shuffle_b200": shuffle_unbatched,
        "naive_shuffle_2_b200": shuffle_naive_batched,
        "shuffle_2_b200": _shuffle_2,
        "shuffle_6_b200": _shuffle_6,
    }
    return types.SimpleNamespace(
        shuffle_batched=shuffle_batched, shuffle_unbatched=shuffle_unbatched,
        shuffle_naive_batched=shuffle_naive_batched, partial_shuffle_batch=partial_shuffle_batch,
        roll_batch=roll_batch, roll_batch_known_threshold=roll_batch_known_threshold,
        roll_batch_naive=roll_batch_naive, digit_pass=digit_pass, ALGORITHMS=algorithms)


# where each bound function lives in the reference package (besides the package namespace)
_HOMES = {
    "shuffle_batched": ("shuffle",), "shuffle_unbatched": ("shuffle",), "shuffle_naive_batched": ("shuffle",),
    "partial_shuffle_batch": ("shuffle",), "roll_batch": ("batched",), "roll_batch_known_threshold": ("batched",),
    "roll_batch_naive": ("batched",), "digit_pass": ("batched",),
}


def register_algorithms(cli, dev=None) -> dict:
    """Add the ``*_b200`` rows to the reference CLI's ``ALGORITHMS`` registry (cli.py:44-49);
    returns the added entries."""
    import importlib

    if dev is None:
        dev = bind(importlib.import_module(cli.__name__.rsplit(".", 1)[0]))
    cli.ALGORITHMS.update(dev.ALGORITHMS)
    return dict(dev.ALGORITHMS)


def install(ref):
    """Route the reference package's hot-path entry points through the device, in place:
    the package namespace and the defining modules (shuffle.py, batched.py); the CLI keeps
    its CPU rows (it imported the originals, cli.py:19-24) and gains the ``*_b200`` rows, so
    ``batchrand bench`` compares the two.  Returns ``uninstall()``."""
    import importlib

    dev = bind(ref)
    saved = []
    mods = {"": ref}
    for sub in ("shuffle", "batched", "cli"):
        try:
            mods[sub] = importlib.import_module(f"{ref.__name__}.{sub}")
        except ImportError:
            pass
    for name, homes in _HOMES.items():
        for where in ("",) + homes:
            m = mods.get(where)
            if m is not None and hasattr(m, name):
                saved.append((m, name, getattr(m, name)))
                setattr(m, name, getattr(dev, name))
    cli = mods.get("cli")
    added = register_algorithms(cli, dev) if cli is not None else {}

    def uninstall():
        for m, name, fn in reversed(saved):
            setattr(m, name, fn)
        if cli is not None:
            for k in added:
                cli.ALGORITHMS.pop(k, None)

    return uninstall


__all__ = ["bind", "install", "register_algorithms"]
