"""Repo-root shim so `import _blockpipe` (the reference's pybind11 module
name, P/python/bindings.cpp:76) resolves to the B200 implementation."""
from paper_2505_21070_b200._blockpipe import *  # noqa: F401,F403
from paper_2505_21070_b200._blockpipe import __all__  # noqa: F401
