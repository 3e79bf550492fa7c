"""Seeded source mutations of oracle functions (test helper): a pin is only trusted if a
plausible mistake in the code it pins makes it fail.  ``mutant(f, old, new)`` returns f
recompiled from its source with the text ``old`` replaced by ``new`` (exactly once)."""
import inspect
import textwrap


def mutant(func, old: str, new: str):
    src = textwrap.dedent(inspect.getsource(func))
    assert src.count(old) == 1, f"mutation site not unique in {func.__name__}: {old!r}"
    src = src.replace(old, new)
    ns = dict(func.__globals__)
    exec(compile(src, f"<mutant of {func.__name__}>", "exec"), ns)
    return ns[func.__name__]
