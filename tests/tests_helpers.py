"""Random program generator shared by CPU and GPU tests (test helper)."""

from paper_2512_23037_b200.circuit import parse_circuit


def random_program(rng, n=None, gates=None, tcount=None, noise_p=None, mpp=True):
    """Random Clifford+T program with noise, M/MR/R, MPP (with flip args),
    feedback (incl. SWAP-controlled), detectors and observables."""
    n = n or rng.choice((2, 3, 5, 8))
    gates = gates or rng.choice((20, 50))
    tcount = rng.choice((2, 6, 10)) if tcount is None else tcount
    noise_p = noise_p if noise_p is not None else rng.choice((0.02, 0.2))
    lines = ["H %d" % rng.randrange(n)]
    meas = 0
    one = ("I", "X", "Y", "Z", "H", "S", "S_DAG", "H_XY", "H_NXY")
    for _ in range(gates):
        r = rng.random()
        if r < 0.12 and tcount > 0:
            tcount -= 1
            lines.append("%s %d" % (rng.choice(("T", "T_DAG")), rng.randrange(n)))
        elif r < 0.40:
            lines.append("%s %d" % (rng.choice(one), rng.randrange(n)))
        elif r < 0.62 and n >= 2:
            a, b = rng.sample(range(n), 2)
            lines.append("%s %d %d" % (rng.choice(("CX", "CZ", "SWAP")), a, b))
        elif r < 0.70:
            lines.append("%s %d" % (rng.choice(("M", "MR", "R")), rng.randrange(n)))
            meas += lines[-1][0] == "M"
        elif r < 0.75 and mpp:
            qs = rng.sample(range(n), min(n, rng.randint(1, 3)))
            prod = "*".join("%s%d" % (rng.choice("XYZ"), q) for q in qs)
            arg = "(%g)" % noise_p if rng.random() < 0.3 else ""
            lines.append("MPP%s %s" % (arg, prod))
            meas += 1
        elif r < 0.84:
            kind = rng.choice(("X_ERROR", "Z_ERROR", "DEPOLARIZE1", "DEPOLARIZE2"))
            if kind == "DEPOLARIZE2" and n >= 2:
                a, b = rng.sample(range(n), 2)
                lines.append("DEPOLARIZE2(%g) %d %d" % (noise_p, a, b))
            else:
                kind = "DEPOLARIZE1" if kind == "DEPOLARIZE2" else kind
                qs = [rng.randrange(n) for _ in range(rng.randint(1, 3))]
                lines.append("%s(%g) %s" % (kind, noise_p, " ".join(map(str, qs))))
        elif r < 0.90 and meas:
            g = rng.choice(("X", "Z", "CX", "CZ", "SWAP"))
            if g == "SWAP":
                lines.append("SWAP rec[-%d] %d" % (rng.randint(1, meas), rng.randrange(n)))
            else:
                lines.append("%s rec[-%d] %d" % (g, rng.randint(1, meas), rng.randrange(n)))
        elif r < 0.95 and meas:
            lines.append("DETECTOR rec[-%d]" % rng.randint(1, meas))
        else:
            lines.append("TICK")
    lines.append("M %d" % rng.randrange(n))
    lines.append("OBSERVABLE_INCLUDE(%d) rec[-1]" % rng.randrange(3))
    return parse_circuit("\n".join(lines) + "\n")
