"""Shared helpers for the test suite (kept out of conftest so test modules can import them)."""


def loop_cases(arrs, tags):
    for t in tags:
        yield t, {k[len(t) + 1:]: v for k, v in arrs.items() if k.startswith(t + "_")}
