"""Loads the CPU oracle (oracle/_build/libsfkv_oracle.so) and the reference shim
(oracle/_ref/libsfref.so). Test infrastructure only."""
import ctypes as C
import os
import subprocess

from paper_2603_13605_b200.abi import Api

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(REPO, "oracle", "_build", "libsfkv_oracle.so")
REF_SO = os.path.join(REPO, "oracle", "_ref", "libsfref.so")
_cache = {}


def load():
    if "oracle" not in _cache:
        src = os.path.join(REPO, "oracle", "sfkv_oracle.c")
        if not os.path.exists(ORACLE_SO) or os.path.getmtime(ORACLE_SO) < os.path.getmtime(src):
            subprocess.run(["make", "-s", "-C", os.path.join(REPO, "oracle")], check=True)
        _cache["oracle"] = Api(C.CDLL(ORACLE_SO), "oracle")
    return _cache["oracle"]


def load_ref():
    """The reference's own functions, or None when oracle/_ref was not built here."""
    if "ref" not in _cache:
        _cache["ref"] = C.CDLL(REF_SO) if os.path.exists(REF_SO) else None
    return _cache["ref"]
