"""Builds paper_2010_16114_b200/variant_dbg.so: the library with -DBS_DEBUG_MODES (the
work-skipping BS_*_MODE switches used by the bound analyses).  On the GPU box, copy it over
libbsb200.so for the experiment: it is never the product library."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2010_16114_b200 import _build as b  # noqa: E402

b.NVCC_FLAGS = b.NVCC_FLAGS + ["-DBS_DEBUG_MODES"]
b.OBJDIR = b.PKG / "build_dbg"
b.LIB = b.PKG / "variant_dbg.so"
print(b.build())
