"""Regenerate tests/golden/rng_ref.json from the REFERENCE's own rng.hpp.

Runs oracle/_ref/rng_ref (built by `make -C oracle ref` from
/root/reference/proj/include/kernid/rng.hpp, unmodified) for a few seeds and
stores its output. Only runnable where /root/reference exists; the JSON is
committed so the pin travels without the reference tree.
"""
import json
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
BIN = os.path.join(ROOT, "oracle", "_ref", "rng_ref")


def main():
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "ref"], check=True)
    out = []
    for seed in (1, 5, 9, 42, 0xDEADBEEF, 2**63 + 12345):
        txt = subprocess.run([BIN, str(seed), "400"], check=True, capture_output=True, text=True).stdout
        out.append(json.loads(txt))
    with open(os.path.join(HERE, "rng_ref.json"), "w") as f:
        json.dump({"source": "oracle/_ref/rng_ref built from /root/reference/proj/include/kernid/rng.hpp",
                   "streams": out}, f)


if __name__ == "__main__":
    main()
