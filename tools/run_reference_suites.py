"""Run the reference's own decoder / renderer / acceptance suites against
this package (tools/refsuite_shim.py): both integration routes, and the
producer route (streams built by the GPU encoder, read by the reference).

    python tools/run_reference_suites.py --stage     # here: copy the tests
    python tools/run_reference_suites.py             # on a GPU box

--stage copies /root/reference/pkg/tests into baseline/_ref/rlfc_tests (git-
ignored, travels to the GPU box with gpurun, like the pip-installed
reference package beside it).  The run writes one JSON summary line per
route and the junit XML under gpurun_out/.
"""
import argparse
import json
import os
import shutil
import subprocess
import sys
import xml.etree.ElementTree as ET

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
TESTS = os.path.join(REF, "rlfc_tests")
SUITES = {
    # Route 1: the public decode/render API and the service on top of it
    "api": ["test_decoder.py", "test_renderer.py", "test_acceptance.py", "test_service.py"],
    # Route 2: everything that reaches the kernel module's decode entry points
    "kernels": ["test_decoder.py", "test_renderer.py", "test_acceptance.py", "test_service.py",
                "test_bise.py", "test_kernels.py"],
    # the producer side: every stream the suites encode comes from the GPU
    # tree construction; the reference decodes and checks them
    "encoder": ["test_encoder.py", "test_decoder.py", "test_container.py", "test_acceptance.py"],
}


def stage():
    src = "/root/reference/pkg/tests"
    if os.path.exists(TESTS):
        shutil.rmtree(TESTS)
    shutil.copytree(src, TESTS, ignore=shutil.ignore_patterns("__pycache__"))
    with open(os.path.join(TESTS, "pytest.ini"), "w") as f:
        f.write("[pytest]\nfilterwarnings =\n    ignore::DeprecationWarning\n    ignore::Warning\n")


def run(route, out_dir):
    env = dict(os.environ, REFSUITE_ROUTE=route,
               PYTHONPATH=os.pathsep.join([REF, ROOT, os.path.join(ROOT, "tools")]))
    xml = os.path.join(out_dir, f"refsuite_{route}.xml")
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "refsuite_shim", "-p", "no:cacheprovider",
           "-c", os.path.join(TESTS, "pytest.ini"), "--rootdir", TESTS, f"--junitxml={xml}"] + \
        [os.path.join(TESTS, s) for s in SUITES[route]]
    p = subprocess.run(cmd, cwd=TESTS, env=env, capture_output=True, text=True)
    tail = p.stdout.strip().splitlines()[-40:]
    res = {"route": route, "rc": p.returncode, "suites": SUITES[route],
           "native_libs": next((ln.split(" ", 1)[1].split(",") for ln in p.stdout.splitlines()
                                if ln.startswith("REFSUITE_NATIVE ")), [])}
    if os.path.exists(xml):
        cases = []
        for tc in ET.parse(xml).getroot().iter("testcase"):
            st = "passed"
            for child in tc:
                if child.tag in ("failure", "error"):
                    st = child.tag
                elif child.tag == "skipped":
                    st = "skipped"
            cases.append((tc.get("classname", "").split(".")[-1] + "::" + tc.get("name"), st))
        res["passed"] = sum(1 for _, s in cases if s == "passed")
        res["failed"] = [n for n, s in cases if s in ("failure", "error")]
        res["skipped"] = [n for n, s in cases if s == "skipped"]
    print(json.dumps(res))
    if p.returncode:
        print("\n".join(tail), file=sys.stderr)
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--stage", action="store_true")
    ap.add_argument("--route", choices=["api", "kernels", "encoder", "all"], default="all")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out"))
    a = ap.parse_args()
    if a.stage:
        stage()
        return
    os.makedirs(a.out, exist_ok=True)
    routes = ["api", "kernels", "encoder"] if a.route == "all" else [a.route]
    for r in routes:
        run(r, a.out)


if __name__ == "__main__":
    main()
