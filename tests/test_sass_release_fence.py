"""Static regression check of the TMA stage-release fix (concurrency
finding): in every TMA-fed kernel of the built library, each consumer release
of a pipeline stage -- the mbarrier arrive on the stage's "empty" barrier --
must be preceded, after the stage's "full" wait, by a cross-proxy fence
(fence.proxy.async, SASS FENCE.VIEW.ASYNC).  Without it the TMA refill can
overtake fragment loads still in flight (profiles/r02_tma_release_race.txt).
compute-sanitizer is not available on the GPU pool, so the property is pinned
on the SASS; runs on the CPU (cuobjdump)."""
import os
import re
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BUILD = os.path.join(ROOT, "paper_2210_12212_b200", "build")


def _functions(obj):
    out = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True, timeout=600).stdout
    name, body = None, []
    for line in out.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            if name:
                yield name, body
            name, body = m.group(1), []
        elif name and re.search(r"/\*[0-9a-f]{4}\*/", line):
            body.append(line.split("*/", 1)[1].split(";")[0].strip())
    if name:
        yield name, body


def _need(obj):
    if shutil.which("cuobjdump") is None:
        pytest.skip("cuobjdump not on PATH")
    path = os.path.join(BUILD, obj)
    if not os.path.exists(path):
        pytest.skip(f"{obj} not built (run __graft_entry__.build())")
    return path


def test_gemm_and_column_pass_release_is_fenced():
    checked = 0
    for obj, pattern in (("gemm_f64.o", "dgemm_tma_kernel"), ("gram_pass.o", "colpass_kernel")):
        for name, body in _functions(_need(obj)):
            if pattern not in name:
                continue
            releases = [i for i, ins in enumerate(body) if "SYNCS.ARRIVE" in ins and ".A1T0" in ins]
            if pattern == "dgemm_tma_kernel":
                assert releases, f"{name}: no consumer release found"
            for i in releases:
                # (the divergent-warp slow path of __syncwarp is laid out of line -- BRA.DIV target,
                # WARPSYNC.COLLECTIVE -- with its own copy of the arrive; it is entered after the fence)
                b = i
                while b > 0 and not (body[b - 1].startswith("BRA ") or body[b - 1].startswith("EXIT")):
                    b -= 1  # (start of the straight-line code that ends in this arrive)
                if any("WARPSYNC.COLLECTIVE" in ins for ins in body[b:i]):
                    continue
                j = i
                while j >= 0 and "SYNCS.PHASECHK" not in body[j]:
                    j -= 1
                assert j >= 0, f"{name}: release without a preceding full-barrier wait"
                window = body[j:i]
                assert any("FENCE.VIEW.ASYNC" in ins for ins in window), (
                    f"{name}: stage released at instruction {i} without a fence.proxy.async after the wait at {j}")
                checked += 1
    assert checked >= 20  # (every TMA GEMM instantiation and both column passes)


def test_dmma_gram_pass_release_is_fenced():
    # gram_dmma_kernel recycles a stage behind a CTA barrier: the fence sits
    # before that barrier, ahead of the refill's UTMALDG.
    found = 0
    for name, body in _functions(_need("gram_pass.o")):
        if "gram_dmma_kernel" not in name:
            continue
        refills = [i for i, ins in enumerate(body) if "UTMALDG" in ins]
        assert refills, f"{name}: no TMA load"
        last_dmma = max(i for i, ins in enumerate(body) if "DMMA" in ins)
        fences = [i for i, ins in enumerate(body) if "FENCE.VIEW.ASYNC" in ins]
        # one fence belongs to the mbarrier set-up; at least one more in the main loop, before a refill
        loop_fences = [i for i in fences if any(r > i for r in refills) and i > min(refills)]
        assert loop_fences, f"{name}: no fence.proxy.async ahead of the stage refill"
        assert min(loop_fences) < last_dmma + 200
        found += 1
    assert found >= 4
