"""`python -m paper_2208_14049_b200.cli` -- the reference's `enserve` CLI
(tools/enserve_cli.cpp: optimize / bench / count / baseline) over the C ABI's
es_cli_main; the commands themselves are C++ (csrc/enserve/commands.cpp)."""
from __future__ import annotations

import ctypes as C
import sys

from ._abi import lib


def main(argv=None) -> int:
    args = [sys.argv[0] if argv is None else "enserve-b200"] + list(sys.argv[1:] if argv is None else argv)
    arr = (C.c_char_p * len(args))(*[a.encode() for a in args])
    sys.stdout.flush()
    return int(lib().es_cli_main(len(args), arr))


if __name__ == "__main__":
    sys.exit(main())
