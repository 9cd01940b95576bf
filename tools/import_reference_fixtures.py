"""Copy the reference's committed golden dumps (data, not code) into
tests/golden/consumer/ so they travel to the GPU box.

Source: /root/reference/pkg/consumer/tests/fixtures/ — produced by the
reference CLI (pkg/scripts/make_consumer_fixtures.py:54-70) and reproduced
bit-exactly by the reference engine in this container.
"""
import os
import shutil

SRC = "/root/reference/pkg/consumer/tests/fixtures"
DST = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                   "tests", "golden", "consumer")

os.makedirs(DST, exist_ok=True)
for name in sorted(os.listdir(SRC)):
    if name.endswith((".json", ".klay")):
        shutil.copyfile(os.path.join(SRC, name), os.path.join(DST, name))
        print("copied", name)
