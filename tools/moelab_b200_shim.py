"""pytest plugin: serve the reference package's `moelab.routing` from the B200 drop-in
(paper_2603_07685_b200.routing) -- the swap INTEGRATION.md describes, applied before the
reference's own tests are collected. Requires the reference installed in baseline/_ref
(bench.py's reference-arm install) on sys.path."""
import sys


def install():
    import moelab

    from paper_2603_07685_b200 import routing as drop_in

    sys.modules["moelab.routing"] = drop_in
    moelab.routing = drop_in
    return drop_in


def pytest_configure(config):
    install()
