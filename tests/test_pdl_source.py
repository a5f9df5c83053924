"""Source invariant of the programmatic dependent launches: a kernel launched with
launch_pdl may start while its predecessor still runs, so its body must open with G2_PDL_WAIT()
(griddepcontrol.wait) before touching memory.  Checked on the CUDA sources, no GPU needed."""
import os
import re

CSRC = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_1811_02761_b200", "csrc")


def sources():
    out = {}
    for f in sorted(os.listdir(CSRC)):
        if f.endswith((".cu", ".cuh")):
            out[f] = open(os.path.join(CSRC, f)).read()
    return out


def kernel_body_start(src, name):
    m = re.search(r"__global__[^;{]*?\b%s\s*\(" % re.escape(name), src, re.S)
    if not m:
        return None
    i = src.index("{", m.end())
    return src[i + 1:i + 400]


def test_every_pdl_launch_waits_first():
    # kernels live in per-file anonymous namespaces (names repeat across files): the launched kernel
    # is the one defined in the launching file
    total = 0
    for f, text in sources().items():
        if f == "common.cuh":  # the helper's own definition
            continue
        for name in sorted(set(re.findall(r"launch_pdl\(\s*([A-Za-z_]\w*)", text))):
            body = kernel_body_start(text, name)
            assert body is not None, (f, name)
            first = body.strip().splitlines()[0]
            assert first.startswith("G2_PDL_WAIT();"), (f, name, first)
            total += 1
    assert total >= 15, total


def test_calc_level_chain_waits_first():
    tree = sources()["tree.cu"]
    for name in ("calc_internal_kernel", "calc_levels_kernel"):
        first = kernel_body_start(tree, name).strip().splitlines()[0]
        assert first.startswith('asm volatile("griddepcontrol.wait;"'), (name, first)
