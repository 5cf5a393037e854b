"""Circuit text front end: Stim-subset grammar plus T/T_DAG.

Host-side API kept for drop-in compatibility with the reference
``gstab.circuit`` (``/root/reference/pkg/src/gstab/circuit.py``):

* ``parse_circuit(text) -> CircuitProgram``   (ref circuit.py:191-205)
* ``CircuitProgram.flat() / serialize() / detectors / observables``
  (ref circuit.py:89-134)
* ``Instruction``, ``Rec``, ``PauliProduct``, ``Block`` value types
  (ref circuit.py:44-86)
* lookback validation and measurement counting (ref circuit.py:340-373)
* ``compute_stats`` (ref circuit.py:392-453), used to report how close the
  MSC proxies come to the paper's Table 2.

Nothing here runs per shot: the program is parsed once and handed to
``compiler.compile_program`` which lowers it to the device op stream.
"""

from __future__ import annotations

import re
from dataclasses import dataclass, field

GATES_1Q = ("I", "X", "Y", "Z", "H", "S", "S_DAG", "H_XY", "H_NXY", "T", "T_DAG")
GATES_2Q = ("CX", "CZ", "SWAP")
NOISE_OPS = ("DEPOLARIZE1", "DEPOLARIZE2", "X_ERROR", "Z_ERROR")
MEASURE_OPS = ("M", "MR", "MPP")
ANNOTATIONS = ("DETECTOR", "OBSERVABLE_INCLUDE", "TICK",
               "QUBIT_COORDS", "SHIFT_COORDS")
FEEDBACK_GATES = ("CX", "CZ", "X", "Z")
KNOWN_OPS = frozenset(GATES_1Q + GATES_2Q + NOISE_OPS + MEASURE_OPS
                      + ANNOTATIONS + ("R",))

_OPCODE = re.compile(r"^([A-Z_0-9]+)(?:\(([^)]*)\))?$")
_LOOKBACK = re.compile(r"^rec\[(-\d+)\]$")
_PRODUCT = re.compile(r"^[XYZ]\d+(?:\*[XYZ]\d+)*$")
_REPEAT = re.compile(r"^REPEAT\s+(\d+)\s*\{$")


class ParseError(ValueError):
    """Parse failure carrying the 1-based line number (ref circuit.py:36-41)."""

    def __init__(self, line_num: int, message: str):
        super().__init__(f"line {line_num}: {message}")
        self.line_num = line_num


@dataclass(frozen=True)
class Rec:
    """Measurement-record lookback ``rec[-k]``; ``offset`` < 0."""
    offset: int

    def __str__(self) -> str:
        return "rec[%d]" % self.offset


@dataclass(frozen=True)
class PauliProduct:
    """MPP target: ((qubit, letter), ...) in the written order."""
    terms: tuple

    def __str__(self) -> str:
        return "*".join("%s%d" % (letter, q) for q, letter in self.terms)

    def qubits(self) -> tuple:
        return tuple(q for q, _ in self.terms)


@dataclass(frozen=True)
class Instruction:
    name: str
    targets: tuple = ()
    args: tuple = ()
    line: int = field(default=0, compare=False, repr=False)

    def __str__(self) -> str:
        head = self.name
        if self.args:
            head += "(" + ", ".join(_format_arg(a) for a in self.args) + ")"
        return " ".join([head] + [str(t) for t in self.targets])


@dataclass(frozen=True)
class Block:
    """``REPEAT count { body }``."""
    count: int
    body: tuple
    line: int = field(default=0, compare=False, repr=False)


def _format_arg(a) -> str:
    f = float(a)
    return str(int(f)) if f == int(f) else repr(f)


def _expand(items):
    for it in items:
        if isinstance(it, Block):
            for _ in range(it.count):
                yield from _expand(it.body)
        else:
            yield it


@dataclass(frozen=True)
class CircuitProgram:
    body: tuple
    num_qubits: int
    num_measurements: int

    def flat(self):
        """Instructions with REPEAT blocks unrolled (ref circuit.py:95-97)."""
        return _expand(self.body)

    def serialize(self) -> str:
        out: list[str] = []

        def emit(items, indent):
            for it in items:
                if isinstance(it, Block):
                    out.append("%sREPEAT %d {" % (indent, it.count))
                    emit(it.body, indent + "    ")
                    out.append(indent + "}")
                else:
                    out.append(indent + str(it))

        emit(self.body, "")
        return "\n".join(out) + "\n"

    def _annotation_indices(self):
        dets, obs, m = [], {}, 0
        for ins in self.flat():
            if ins.name in MEASURE_OPS:
                m += len(ins.targets)
            elif ins.name == "DETECTOR":
                dets.append(tuple(m + t.offset for t in ins.targets))
            elif ins.name == "OBSERVABLE_INCLUDE":
                key = int(ins.args[0]) if ins.args else 0
                obs.setdefault(key, []).extend(m + t.offset for t in ins.targets)
        return dets, obs

    @property
    def detectors(self) -> list:
        """Absolute record indices per detector, execution order."""
        return self._annotation_indices()[0]

    @property
    def observables(self) -> dict:
        obs = self._annotation_indices()[1]
        return {k: tuple(sorted(v)) for k, v in obs.items()}

    def has_noise(self) -> bool:
        return any(i.name in NOISE_OPS or (i.name == "MPP" and i.args)
                   for i in self.flat())


# ----------------------------------------------------------------------
# parsing
# ----------------------------------------------------------------------

def parse_circuit(text: str) -> CircuitProgram:
    """Parse circuit text; qubit count = 1 + max target (ref circuit.py:191)."""
    lines = text.splitlines()
    body, _ = _parse_lines(lines, 0, nested=False)
    body = tuple(body)
    top = -1
    for ins in _expand(body):
        for t in ins.targets:
            if isinstance(t, int):
                top = max(top, t)
            elif isinstance(t, PauliProduct):
                top = max(top, *t.qubits())
    return CircuitProgram(body=body, num_qubits=top + 1,
                          num_measurements=_check_lookbacks(body))


def _parse_lines(lines, pos, nested):
    body = []
    while pos < len(lines):
        text = lines[pos].split("#", 1)[0].strip()
        lineno = pos + 1
        if not text:
            pos += 1
            continue
        if text == "}":
            if not nested:
                raise ParseError(lineno, "unbalanced '}'")
            return body, pos + 1
        if text.startswith("REPEAT"):
            m = _REPEAT.match(text)
            if m is None:
                raise ParseError(lineno, "malformed REPEAT header "
                                 "(expected 'REPEAT n {')")
            count = int(m.group(1))
            if count < 1:
                raise ParseError(lineno, "REPEAT count must be >= 1")
            inner, pos = _parse_lines(lines, pos + 1, nested=True)
            body.append(Block(count=count, body=tuple(inner), line=lineno))
            continue
        body.append(_parse_one(text, lineno))
        pos += 1
    if nested:
        raise ParseError(len(lines), "unbalanced '{': block never closed")
    return body, pos


def _parse_one(text: str, lineno: int) -> Instruction:
    words = text.split()
    m = _OPCODE.match(words[0])
    if m is None:
        raise ParseError(lineno, "malformed opcode %r" % words[0])
    name = m.group(1)
    if name not in KNOWN_OPS:
        raise ParseError(lineno, "unknown opcode %r" % name)
    args = ()
    if m.group(2) is not None:
        try:
            args = tuple(float(a) for a in m.group(2).split(",") if a.strip())
        except ValueError:
            raise ParseError(lineno, "malformed arguments in %r" % words[0])
    targets = tuple(_parse_target(w, name, lineno) for w in words[1:])
    _validate_shape(name, targets, args, lineno)
    return Instruction(name=name, targets=targets, args=args, line=lineno)


def _parse_target(word: str, opcode: str, lineno: int):
    m = _LOOKBACK.match(word)
    if m is not None:
        off = int(m.group(1))
        if off >= 0:
            raise ParseError(lineno, "lookback must be negative: %s" % word)
        return Rec(off)
    if word.isdigit():
        return int(word)
    if opcode == "MPP" and _PRODUCT.match(word):
        terms = tuple((int(a[1:]), a[0]) for a in word.split("*"))
        if len({q for q, _ in terms}) != len(terms):
            raise ParseError(lineno, "repeated qubit in product %r" % word)
        return PauliProduct(terms=terms)
    raise ParseError(lineno, "malformed target %r" % word)


def _pairs(seq):
    it = iter(seq)
    return list(zip(it, it))


def _validate_shape(name, targets, args, lineno):
    """Per-opcode target/argument rules (ref circuit.py:278-332)."""
    n_rec = sum(isinstance(t, Rec) for t in targets)
    n_prod = sum(isinstance(t, PauliProduct) for t in targets)
    if name in ("TICK", "SHIFT_COORDS"):
        if targets:
            raise ParseError(lineno, "%s takes no targets" % name)
        return
    if name in ("DETECTOR", "OBSERVABLE_INCLUDE"):
        if n_rec != len(targets):
            raise ParseError(lineno, "%s targets must be lookbacks" % name)
        return
    if name == "QUBIT_COORDS":
        if len(targets) != 1 or not isinstance(targets[0], int):
            raise ParseError(lineno, "QUBIT_COORDS takes one qubit target")
        return
    if name == "MPP":
        if not targets or n_prod != len(targets):
            raise ParseError(lineno, "MPP targets must be Pauli products")
        return
    if n_prod:
        raise ParseError(lineno, "%s cannot take Pauli products" % name)
    if name in NOISE_OPS:
        if len(args) != 1 or not 0.0 <= args[0] <= 1.0:
            raise ParseError(lineno, "%s needs one probability argument" % name)
        if n_rec:
            raise ParseError(lineno, "%s targets must be qubits" % name)
        if name == "DEPOLARIZE2":
            if not targets or len(targets) % 2:
                raise ParseError(lineno, "DEPOLARIZE2 needs qubit pairs")
        elif not targets:
            raise ParseError(lineno, "%s needs at least one target" % name)
        return
    if not targets:
        raise ParseError(lineno, "%s needs targets" % name)
    if name in GATES_2Q:
        if len(targets) % 2:
            raise ParseError(lineno, "%s needs target pairs" % name)
        for a, b in _pairs(targets):
            if isinstance(b, Rec):
                raise ParseError(lineno, "lookback allowed only as a control")
            if isinstance(a, int) and a == b:
                raise ParseError(lineno, "duplicate target %d" % a)
        return
    if name in ("X", "Z") and n_rec:
        if len(targets) % 2 or any(
                not isinstance(a, Rec) or not isinstance(b, int)
                for a, b in _pairs(targets)):
            raise ParseError(lineno,
                             "conditional %s needs (rec, qubit) pairs" % name)
        return
    if n_rec:
        raise ParseError(lineno, "%s targets must be qubits" % name)


def _check_lookbacks(body) -> int:
    """Validate that every lookback resolves at its first execution and
    return the total measurement count (ref circuit.py:340-373)."""

    def walk(items, m):
        for it in items:
            if isinstance(it, Block):
                after = walk(it.body, m)
                m += it.count * (after - m)
                continue
            for t in it.targets:
                if isinstance(t, Rec) and -t.offset > m:
                    raise ParseError(
                        it.line, "lookback %s resolves before any of the %d "
                        "measurements made so far" % (t, m))
            if it.name in MEASURE_OPS:
                m += len(it.targets)
        return m

    return walk(body, 0)


def resolve_detector(lookbacks, record) -> int:
    """XOR of the referenced record bits (ref circuit.py:380-389)."""
    parity = 0
    for lb in lookbacks:
        k = lb.offset if isinstance(lb, Rec) else int(lb)
        if k >= 0 or -k > len(record):
            raise IndexError("lookback %d out of range for record of length %d"
                             % (k, len(record)))
        parity ^= record[k]
    return parity


# ----------------------------------------------------------------------
# statistics (Table 2 columns)
# ----------------------------------------------------------------------

@dataclass(frozen=True)
class CircuitStats:
    total_qubits: int
    total_gates: int
    depth: int
    two_qubit_gates: int
    measurements: int
    t_count: int
    t_support_size: int
    t_depth: int

    def as_dict(self) -> dict:
        return dict(self.__dict__)


def compute_stats(prog) -> CircuitStats:
    """Gate/measurement/T statistics; noise, annotations and feedback are not
    gates; depth counts TICK layers with activity (ref circuit.py:392-453)."""
    g1 = g2 = meas = tcount = depth = tdepth = 0
    support: set = set()
    active = has_t = False
    for ins in prog.flat():
        name = ins.name
        if name == "TICK":
            if active:
                depth += 1
                tdepth += has_t
            active = has_t = False
            continue
        if name in NOISE_OPS or name in ANNOTATIONS:
            continue
        if any(isinstance(t, Rec) for t in ins.targets):
            continue
        if name in GATES_2Q:
            g2 += len(ins.targets) // 2
        elif name in ("T", "T_DAG"):
            tcount += len(ins.targets)
            support.update(ins.targets)
            g1 += len(ins.targets)
            has_t = True
        elif name in GATES_1Q:
            g1 += len(ins.targets)
        elif name in MEASURE_OPS:
            meas += len(ins.targets)
        elif name != "R":
            continue
        active = True
    if active:
        depth += 1
        tdepth += has_t
    return CircuitStats(prog.num_qubits, g1 + g2, depth, g2, meas, tcount,
                        len(support), tdepth)
