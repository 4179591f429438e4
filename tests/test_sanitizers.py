"""Host code under AddressSanitizer + UndefinedBehaviorSanitizer (host ASan/UBSan): the
oracle (every entry point on small, partly malformed inputs) and the library's GPU-free host paths,
each in a subprocess that preloads the sanitizer runtimes; any report fails the test. (Device-side
compute-sanitizer is not available on this pool's GPU boxes.)"""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _runtime(name):
    p = subprocess.run(["gcc", f"-print-file-name={name}"], capture_output=True, text=True).stdout.strip()
    return p if os.path.isabs(p) and os.path.exists(p) else None


def test_oracle_clean_under_asan_ubsan(tmp_path):
    asan, ubsan = _runtime("libasan.so"), _runtime("libubsan.so")
    if not asan or not ubsan:
        pytest.skip("sanitizer runtimes not installed")
    so = tmp_path / "liboracle_san.so"
    subprocess.check_call(["gcc", "-O1", "-g", "-fsanitize=address,undefined", "-fno-omit-frame-pointer",
                           "-std=c11", "-fPIC", "-shared", "-pthread", "-o", str(so),
                           os.path.join(ROOT, "oracle", "dip_oracle.c"), "-lm"])
    env = dict(os.environ, LD_PRELOAD=f"{asan}:{ubsan}", ASAN_OPTIONS="detect_leaks=0",
               UBSAN_OPTIONS="print_stacktrace=1", ORACLE_LIB=str(so), PYTHONPATH=ROOT)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "scripts", "oracle_workout.py")],
                         capture_output=True, text=True, env=env, timeout=600, cwd=ROOT)
    log = out.stdout + out.stderr
    assert out.returncode == 0, log[-3000:]
    assert "AddressSanitizer" not in log and "runtime error" not in log, log[-3000:]
    assert "done" in out.stdout


def test_library_host_code_clean_under_asan_ubsan(tmp_path):
    # the product's host-side code paths that run without a GPU (model loading and its guards, record
    # encoding, plan compilation and the discrete-event plan validator) from a sanitizer build of
    # libdip, through the same boundary / plan tests as the regular build
    asan, ubsan = _runtime("libasan.so"), _runtime("libubsan.so")
    if not asan or not ubsan:
        pytest.skip("sanitizer runtimes not installed")
    sys.path.insert(0, ROOT)
    from paper_2504_14145_b200 import build as B
    inc, lib = B._nccl_dirs()
    so = tmp_path / "libdip_san.so"
    cmd = [B.NVCC, "-O1", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a",
           "-Xcompiler", "-fPIC,-fsanitize=address,-fsanitize=undefined,-fno-omit-frame-pointer", "-shared",
           "-I", os.path.join(ROOT, "include"), "-I", os.path.join(B.HERE, "csrc"), *B.SRCS, "-o", str(so)]
    if inc:
        cmd[1:1] = ["-I", inc]
        cmd += ["-L", lib, "-l:libnccl.so.2", "-Xlinker", f"-rpath={lib}"]
    else:
        cmd += ["-lnccl"]
    subprocess.check_call(cmd)
    env = dict(os.environ, LD_PRELOAD=f"{asan}:{ubsan}", ASAN_OPTIONS="detect_leaks=0:protect_shadow_gap=0",
               DIP_LIB=str(so), PYTHONPATH=ROOT)
    out = subprocess.run([sys.executable, "-m", "pytest", "-q", "-s", "-p", "no:cacheprovider",
                          os.path.join(ROOT, "tests", "test_boundary.py"), os.path.join(ROOT, "tests", "test_plan.py")],
                         capture_output=True, text=True, env=env, timeout=900, cwd=ROOT)
    log = out.stdout + out.stderr
    assert out.returncode == 0, log[-3000:]
    assert "AddressSanitizer" not in log and "runtime error" not in log, log[-3000:]
