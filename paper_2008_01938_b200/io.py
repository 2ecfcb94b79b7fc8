"""Instance text I/O and split-table parenthesisation (host logic).

Mirrors include/pipedp/io.hpp (the reference's io.hpp:14-31 / io.cpp:10-80
formats) for Python callers: `sdp n k opname / offsets / init` and
`mcm n / dims`, a batched loader (every instance in a file, in order -- the
input side of solve_sequential_batch / solve_mcm_batch) and the optimal
parenthesisation from solve_mcm_with_split's split table."""
from typing import List, Sequence, Union

from . import OPS, Error, McmInstance, SdpInstance, cell_count, lin, validate

Instance = Union[SdpInstance, McmInstance]


def to_text(inst: Instance) -> str:
    """to_text (io.cpp:30-42): bit-exact round trip with read_instance."""
    if isinstance(inst, SdpInstance):
        return (f"sdp {inst.n} {len(inst.offsets)} {inst.op}\n" + " ".join(str(int(v)) for v in inst.offsets) +
                "\n" + " ".join(str(int(v)) for v in inst.init) + "\n")
    return f"mcm {inst.n}\n" + " ".join(str(int(v)) for v in inst.dims) + "\n"


def _ints(tokens, count, what):
    out = []
    for _ in range(count):
        try:
            out.append(int(next(tokens)))
        except (StopIteration, ValueError):
            raise Error(11, f"InvalidParams: malformed instance: missing {what}") from None
    return out


def _parse(header, tokens) -> Instance:
    if header == "sdp":
        n, k = _ints(tokens, 1, "n")[0], _ints(tokens, 1, "k")[0]
        try:
            op = next(tokens)
        except StopIteration:
            raise Error(11, "InvalidParams: malformed instance: missing operator name") from None
        if op not in OPS:
            raise Error(11, f"InvalidParams: unknown operator name: {op}")
        offs = _ints(tokens, k, "offset")
        init = _ints(tokens, offs[0] if offs else 0, "initial value")
        return validate(SdpInstance(n, offs, init, op))
    if header == "mcm":
        n = _ints(tokens, 1, "n")[0]
        return validate(McmInstance(_ints(tokens, n + 1, "dimension")))
    raise Error(11, f"InvalidParams: unknown instance header: {header}")


def read_instances(text: str) -> List[Instance]:
    """Every instance in `text`, in order (validated; Error on malformed input)."""
    tokens = iter(text.split())
    out = [_parse(h, tokens) for h in tokens]
    if not out:
        raise Error(11, "InvalidParams: empty instance file")
    return out


def read_instance(text: str) -> Instance:
    """read_instance (io.cpp:56-80): the first instance in `text`."""
    tokens = iter(text.split())
    for h in tokens:
        return _parse(h, tokens)
    raise Error(11, "InvalidParams: empty instance file")


def read_instance_file(path: str) -> Instance:
    try:
        return read_instance(open(path).read())
    except OSError:
        raise Error(11, f"InvalidParams: cannot open instance file: {path}") from None


def read_instances_file(path: str) -> List[Instance]:
    try:
        return read_instances(open(path).read())
    except OSError:
        raise Error(11, f"InvalidParams: cannot open instance file: {path}") from None


def mcm_parenthesization(dims: Sequence[int], split: Sequence[int]) -> str:
    """Optimal parenthesisation "((A1A2)A3)" from a split table (reference
    layout, 1-based term index per cell; mcm.cpp:105)."""
    n = len(dims) - 1
    if n < 1 or len(split) != cell_count(n) + 1:
        raise Error(11, "InvalidParams: split table size != n(n+1)/2 + 1")
    out = []
    stack = [(1, n, 0)]
    while stack:
        r, c, state = stack.pop()
        if r == c:
            out.append(f"A{r}")
            continue
        j = int(split[lin(r, c, n)])
        if not 1 <= j <= c - r:
            raise Error(11, "InvalidParams: split index out of range")
        k = r + j - 1
        if state == 0:
            out.append("(")
            stack += [(r, c, 2), (k + 1, c, 0), (r, k, 0)]
        else:
            out.append(")")
    return "".join(out)
