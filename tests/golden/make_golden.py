"""Freeze the reference's own outcomes for the transport scenarios (SPEC known-answer examples
+ seeded random schedules) into spec_examples.json, by running the UNMODIFIED reference fanpipe
(baseline/_ref, pip-installed from /root/reference/pkg). Re-run after rebuilding baseline/_ref:

    python tests/golden/make_golden.py
"""

import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, os.path.dirname(HERE))

from transport_schedules import RefAdapter, random_scenario, run, spec_scenarios  # noqa: E402


def main():
    scen = dict(spec_scenarios())
    scen["random_latest_s1"] = random_scenario(1, "latest", 5, 3)
    scen["random_latest_s2_cap2"] = random_scenario(2, "latest", 2, 3)
    scen["random_fifo_s3"] = random_scenario(3, "fifo", 4, 2)
    out = {}
    for name, sc in scen.items():
        out[name] = {"scenario": sc, "outcomes": run(RefAdapter(), sc)}
    with open(os.path.join(HERE, "spec_examples.json"), "w") as f:
        json.dump(out, f, indent=None, separators=(",", ":"))
    print(f"wrote {len(out)} scenarios")


if __name__ == "__main__":
    main()
