"""Generates tests/golden/ref_fixtures.json by running the REFERENCE engine
(oracle/_ref/ref_snapshot: the unmodified reference library built from
/root/reference) on every case of cases.py. Run in the build container:

    make -C oracle ref && python tests/golden/make_fixtures.py
"""
import json
import os
import shutil
import subprocess
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, HERE)
from cases import all_cases  # noqa: E402

DRIVER = os.path.join(ROOT, "oracle", "_ref", "ref_snapshot")


def main():
    out = {"generator": "oracle/_ref/ref_snapshot (reference engine, unthrottled, chunk 64 KiB, no fsync)",
           "cases": {}}
    tmp = tempfile.mkdtemp(prefix="lzk_fix_")
    try:
        for w, thr in all_cases():
            spec = w.write_spec(os.path.join(tmp, w.name + ".spec"))
            root = os.path.join(tmp, w.name)
            r = subprocess.run([DRIVER, "--spec", spec, "--root", root, "--threshold", str(thr), "--chunk",
                                str(64 << 10), "--restore", "1"], check=True, capture_output=True, text=True)
            res = json.loads(r.stdout)
            rank = res["ranks"][0]
            assert rank["restore_exact"], w.name
            out["cases"][w.name] = {"threshold": thr, "payload": rank["steps"][0]["payload"],
                                    "files": {f["path"]: {"size": f["size"], "fnv": f["fnv"]} for f in rank["files"]}}
            print(w.name, out["cases"][w.name]["files"])
    finally:
        shutil.rmtree(tmp, ignore_errors=True)
    with open(os.path.join(HERE, "ref_fixtures.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
