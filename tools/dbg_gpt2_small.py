"""Debug driver: `bench.py --config gpt2` with a modified GPT-2 shape
(DBG_LAYERS, DBG_SEQ, DBG_VOCAB env vars)."""
import dataclasses
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_16028_b200 import lowerings as L  # noqa: E402

L.GPT2_SMALL = dataclasses.replace(L.GPT2_SMALL, layers=int(os.environ.get("DBG_LAYERS", "12")),
                                   seq=int(os.environ.get("DBG_SEQ", "1024")),
                                   vocab=int(os.environ.get("DBG_VOCAB", "50257")),
                                   act=os.environ.get("DBG_ACT", "gelu"),
                                   bias=os.environ.get("DBG_BIAS", "1") == "1",
                                   norm=os.environ.get("DBG_NORM", "ln"))
import bench  # noqa: E402

bench.main(["--config", "gpt2", "--no-cpu"] + sys.argv[1:])
