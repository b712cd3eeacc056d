"""Validation messages and automatic near-grid sizes produced by the REFERENCE
(`perisum.model.validate_problem`, model.py:211-297; `auto_near_dims`,
model.py:146-162) on the seeded problems of validation_cases.py.

Run in the build container (where /root/reference exists):
    python tests/golden/make_validation_golden.py
Writes validation_golden.json (committed); tests/test_problem_cpu.py compares
this repo's host-side validation against it message for message.  Nothing at
run time reads /root/reference.
"""
from __future__ import annotations

import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, HERE)


def main():
    import perisum.model as ref
    import validation_cases as vc

    out = {"messages": {}, "auto_near_dims": []}
    for name in vc.CASES:
        cfg, box, src, obs, params = vc.build(name, ref)
        out["messages"][name] = list(ref.validate_problem(cfg, box, src, obs, params).messages)
    for n, d in vc.AUTO_DIMS:
        out["auto_near_dims"].append([n, list(d), list(ref.auto_near_dims(n, ref.TargetBox(d)))])
    path = os.path.join(HERE, "validation_golden.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    n_msg = sum(len(v) for v in out["messages"].values())
    print(f"wrote {path}: {len(out['messages'])} cases, {n_msg} messages, {len(out['auto_near_dims'])} grid sizes")


if __name__ == "__main__":
    main()
