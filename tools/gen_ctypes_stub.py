"""Generate the ctypes mirror of include/leafi_b200.h's structs for INTEGRATION.md.

    python tools/gen_ctypes_stub.py            # print the stub
    python tools/gen_ctypes_stub.py --write    # refresh the block in INTEGRATION.md

tests/test_lib_cpu.py checks that INTEGRATION.md carries exactly this output,
so the documented binding cannot drift from the header."""

import re
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "leafi_b200.h"
DOC = ROOT / "INTEGRATION.md"
BEGIN, END = "<!-- ctypes-stub:begin (tools/gen_ctypes_stub.py) -->", "<!-- ctypes-stub:end -->"
CTYPE = {"int64_t": "C.c_int64", "int32_t": "C.c_int32", "double": "C.c_double", "int": "C.c_int"}
CLASSES = {"lf_index": "LfIndex", "lf_search_opts": "LfSearchOpts", "lf_trace": "LfTrace"}


def struct_fields(text: str, name: str) -> list:
    body = re.search(r"typedef struct %s \{(.*?)\} %s;" % (name, name), text, re.S).group(1)
    body = re.sub(r"/\*.*?\*/", "", body, flags=re.S)
    out = []
    for decl in (d.strip() for d in body.split(";")):
        if not decl:
            continue
        m = re.match(r"(const\s+)?(\w+)\s*(\*?)\s*(\w+)\s*(\[(\w+)\])?$", decl)
        typ, ptr, field, dim = m.group(2), m.group(3), m.group(4), m.group(6)
        ct = "C.c_void_p" if ptr else CTYPE[typ]
        if dim:
            ct = f"{ct} * {dim}"
        out.append((field, ct))
    return out


def stub() -> str:
    text = HEADER.read_text()
    lines = ["```python", "import ctypes as C", "", "LF_MAX_SEG = 64", ""]
    for cname, pyname in CLASSES.items():
        lines.append(f"class {pyname}(C.Structure):                # include/leafi_b200.h: {cname}")
        lines.append("    _fields_ = [")
        for f, ct in struct_fields(text, cname):
            lines.append(f'        ("{f}", {ct.replace("LF_MAX_SEG", "LF_MAX_SEG")}),')
        lines.append("    ]")
        lines.append("")
    lines += [
        "lib = C.CDLL(\"libleafi_b200.so\")",
        "lib.lf_last_error.restype = C.c_char_p",
        "lib.lf_abi_sizeof.restype = C.c_int64",
        "lib.lf_abi_offsetof.restype = C.c_int64",
        "for _name, _cls in ((\"lf_index\", LfIndex), (\"lf_search_opts\", LfSearchOpts), (\"lf_trace\", LfTrace)):",
        "    assert lib.lf_abi_sizeof(_name.encode()) == C.sizeof(_cls), _name      # layout check at load",
        "    for _f, _ in _cls._fields_:",
        "        assert lib.lf_abi_offsetof(_name.encode(), _f.encode()) == getattr(_cls, _f).offset, (_name, _f)",
        "```",
    ]
    return "\n".join(lines)


def doc_block() -> str:
    return f"{BEGIN}\n{stub()}\n{END}"


if __name__ == "__main__":
    if "--write" in sys.argv:
        d = DOC.read_text()
        a, b = d.index(BEGIN), d.index(END) + len(END)
        DOC.write_text(d[:a] + doc_block() + d[b:])
    else:
        print(stub())
