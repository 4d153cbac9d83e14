"""Regenerates tests/golden/kat_config_a.json (SURVEY §8c digest recipe) from the
compiled reference (oracle/_ref) — run in the build container, where
/root/reference exists.  The committed JSON is what the tests compare against."""
import json
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
from tests.kat import config_a_digest  # noqa: E402

if __name__ == "__main__":
    out = {name: config_a_digest("ref", name) for name in ("exec_only", "mm_exec")}
    path = os.path.join(os.path.dirname(__file__), "kat_config_a.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)
    print(json.dumps(out, indent=1))
