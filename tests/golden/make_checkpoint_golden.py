"""Writes tests/golden/ckpt_ref.wssr with the REFERENCE's own checkpoint writer
(vmcsr/checkpoint.py, imported read-only from /root/reference) on the inputs of
tests/test_checkpoint.py::golden_inputs, so the drop-in's reader/writer is pinned to real
reference bytes.  Run in the build container: python tests/golden/make_checkpoint_golden.py"""
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")

from vmcsr import checkpoint as ref_ckpt  # noqa: E402

from test_checkpoint import golden_inputs  # noqa: E402

scalars, arrays, rngs = golden_inputs()
ref_ckpt.write_checkpoint(os.path.join(HERE, "ckpt_ref.wssr"), scalars, arrays, rngs)
print("wrote", os.path.join(HERE, "ckpt_ref.wssr"))
