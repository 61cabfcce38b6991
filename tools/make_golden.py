"""Generate tests/golden/*.json — small known-answer vectors for the product
path, with their expected results computed by Python's exact integer
arithmetic and cross-checked against GMP (oracle/port.py).

    python tools/make_golden.py

Inputs follow the reference generator's kinds (gen_inputs.cpp:10-100):
uniform words from std::mt19937_64, the STRUCTURED boundary list, and the
ADVERSARIAL chunk patterns near the balanced-split boundary.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import port  # noqa: E402


def structured_values(n):
    """gen_inputs.cpp:23-46."""
    vals = []

    def push(v):
        v &= (1 << n) - 1
        if v not in vals:
            vals.append(v)

    push(0)
    push(1)
    push(2)
    push(3)
    push(1 << (n // 2))
    push(1 << (n - 1))
    push((1 << (n - 1)) + 1)
    push((1 << (n - 1)) - 1)
    push((1 << n) - 1)
    push((1 << n) - 2)
    push(int("5" * ((n + 3) // 4), 16))
    push(int("a" * ((n + 3) // 4), 16))
    return vals


def adversarial_value(words, n, b):
    """Chunks near the balanced boundary 2^(b-1) (gen_inputs.cpp:48-68),
    driven by the given mt19937_64 words."""
    chunks = (n + b - 1) // b
    v = 0
    for i in range(chunks):
        eta = int(words[i % len(words)]) % 4
        chunk = max(0, (1 << (b - 1)) - 2 + eta)
        v = (v << b) + chunk
    return v & ((1 << n) - 1)


def uniform_value(seed, n):
    nl = (n + 63) // 64
    w = port.mt19937_64(seed, nl)
    return port.limbs_to_int(w) & ((1 << n) - 1)


def entry(n, u, v, tag):
    p = u * v
    nl = (n + 63) // 64
    ul = port.int_to_limbs(u, nl)
    vl = port.int_to_limbs(v, nl)
    assert port.limbs_to_int(port.gmp_mul(ul, vl)) == p, "GMP disagrees with Python"
    hs = [p >> n]
    if p & ((1 << n) - 1) and (p >> n) + 1 <= (1 << n):
        hs.append((p >> n) + 1)
    return {"tag": tag, "n": n, "u": format(u, "x"), "v": format(v, "x"),
            "full": format(p, "x"), "low": format(p & ((1 << n) - 1), "x"),
            "high_set": [format(h, "x") for h in hs]}


def main():
    out = []
    for n in (4095, 4096, 5001, 8192, 20011):
        for s in range(3):
            out.append(entry(n, uniform_value(1000 + 17 * n + s, n),
                             uniform_value(2000 + 17 * n + s, n), f"uniform-{s}"))
        if n > 8192:
            continue
        sv = structured_values(n)
        for i, a in enumerate(sv):
            b_ = sv[(i * 5 + 3) % len(sv)]
            out.append(entry(n, a, b_, f"structured-{i}"))
            out.append(entry(n, a, a, f"structured-sq-{i}"))
        words = port.mt19937_64(77 + n, 64)
        for bb in (12, 13, 14, 15):
            out.append(entry(n, adversarial_value(words, n, bb),
                             adversarial_value(words[::-1], n, bb), f"adversarial-b{bb}"))
    # reference CLI examples (SPEC.md cli section: mul 3 3 -> 9,
    # mulhi --n 12 fff fff -> ffe or fff).  SPEC.md also lists
    # "mullo --n 12 abc def -> 894", which is arithmetically wrong:
    # 0xabc * 0xdef = 0x959184, whose low 12 bits are 0x184 -- the value the
    # reference's own oracle_low (oracle.cpp) and low_product return.
    cli = [
        {"cmd": "mullo", "n": 12, "u": "abc", "v": "def", "expect": ["184"]},
        {"cmd": "mul", "n": 2, "u": "3", "v": "3", "expect": ["9"]},
        {"cmd": "mulhi", "n": 12, "u": "fff", "v": "fff", "expect": ["ffe", "fff"]},
    ]
    for c in cli:
        u, v, n = int(c["u"], 16), int(c["v"], 16), c["n"]
        if c["cmd"] == "mullo":
            assert format((u * v) & ((1 << n) - 1), "x") in c["expect"]
        elif c["cmd"] == "mul":
            assert format(u * v, "x") in c["expect"]
    # parameter pins of the reference tests (test_products.cpp:179-215)
    params = {
        "reference_1e6": {
            "low": {"b": 14, "N": 71680, "lambda": 4, "p": 65},
            "high": {"b": 14, "N": 71680, "lambda": 4, "p": 68},
            "full": {"b": 21, "N": 49152, "lambda": 0, "p": 60},
        },
        "fallback": [
            {"n": 4095, "mode": "low", "backend": "fft", "cutoff": 4096, "mode_out": "fallback"},
            {"n": 4096, "mode": "low", "backend": "exact", "cutoff": 4096, "mode_out": "low"},
            {"n": 99, "mode": "full", "backend": "exact", "cutoff": 100, "mode_out": "fallback"},
            {"n": 100, "mode": "full", "backend": "exact", "cutoff": 100, "mode_out": "full"},
        ],
        "tiny_exact": {"n": 12, "mode": "low", "b": 4, "N": 3, "p": 20},
    }
    os.makedirs(os.path.join(ROOT, "tests", "golden"), exist_ok=True)
    with open(os.path.join(ROOT, "tests", "golden", "products.json"), "w") as f:
        json.dump({"generator": "tools/make_golden.py", "vectors": out, "cli": cli}, f, indent=0)
    with open(os.path.join(ROOT, "tests", "golden", "params.json"), "w") as f:
        json.dump(params, f, indent=1)
    print(f"wrote {len(out)} vectors")


if __name__ == "__main__":
    main()
