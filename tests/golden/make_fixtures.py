"""Regenerates tests/golden/fixtures/*.json from the reference's bundled
fixtures (/root/reference/proj/fixtures, read-only, not present on the GPU
box): each document is parsed by this repo's feeder reader and re-emitted by
its serializer (sorted keys, 2-space layout), then checked to round-trip to an
identical feeder. Run in the build container:  python tests/golden/make_fixtures.py
"""
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from paper_2501_08293_b200 import dopf  # noqa: E402

SRC = "/root/reference/proj/fixtures"
NAMES = ["single_bus", "two_bus", "three_bus_transformer", "four_bus_delta", "two_bus_delta"]

if __name__ == "__main__":
    os.makedirs(os.path.join(HERE, "fixtures"), exist_ok=True)
    for name in NAMES:
        f = dopf.parse_feeder_file(os.path.join(SRC, name + ".json"))
        text = f.serialize()
        again = dopf.parse_feeder(text)
        assert again.serialize() == text, name
        with open(os.path.join(HERE, "fixtures", name + ".json"), "w") as out:
            out.write(text + "\n")
        print("wrote", name)
