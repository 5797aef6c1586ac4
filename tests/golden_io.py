"""Readers for the cited text fixtures under tests/golden/."""
import os

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _lines(name):
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.strip()
            if line and not line.startswith("#"):
                yield line.split()


def rows_and_cases(name):
    """(rows, cases, status) of a single-block policy fixture."""
    rows, cases, status = [], [], None
    for tok in _lines(name):
        if tok[0] == "row":
            rows.append(tuple(int(t) for t in tok[1:7]))
        elif tok[0] == "case":
            cases.append(tuple(t if t == "default" else int(t) for t in tok[1:]))
        elif tok[0] == "status":
            status = tok[1]
    return rows, cases, status


def blocks(name):
    """{block_name: (rows, cases)} of a multi-block policy fixture."""
    out, cur = {}, None
    for tok in _lines(name):
        if tok[0] == "block":
            cur = tok[1]
            out[cur] = ([], [])
        elif tok[0] == "end":
            cur = None
        elif tok[0] == "row":
            out[cur][0].append(tuple(int(t) for t in tok[1:7]))
        elif tok[0] == "case":
            out[cur][1].append(tuple(t if t == "default" else int(t) for t in tok[1:]))
    return out


def table(name):
    return [tuple(float(t) for t in tok) for tok in _lines(name)]
