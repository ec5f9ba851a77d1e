"""Regenerate tests/golden/rng_reference.json from the REFERENCE's own rng.hpp.

oracle/Makefile's `ref` target compiles oracle/ref_rng_dump.cpp against
/root/reference/proj/include/lmra/rng.hpp (the only Eigen-free file on the hot path)
into oracle/_ref/ref_rng_dump; its JSON output is committed here so the GPU box (which
has no /root/reference) and the CPU tests can pin the oracle and the product's host
RNG against the reference itself.

    python tests/golden/make_golden.py
"""
import json
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))


def main():
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "ref"], check=True)
    out = subprocess.run([os.path.join(ROOT, "oracle", "_ref", "ref_rng_dump")], check=True,
                         capture_output=True, text=True).stdout
    data = json.loads(out)
    with open(os.path.join(HERE, "rng_reference.json"), "w") as f:
        json.dump(data, f, indent=1)
    print("wrote", len(data["streams"]), "streams")


if __name__ == "__main__":
    main()
