"""Report / pipeline / CLI layer and metrics (§8 f4).

tests/cpp/pipeline_kats.cpp restates the reference's pipeline, mesh-I/O and
metrics tests (proj/tests/pipeline_tests.cpp, mesh_io_tests.cpp,
metrics_tests.cpp): its "cpu:" cases (JSON format, files, metrics, validation)
run here; its "gpu:" cases run the whole pipeline, i.e. the MM loop on the
B200. The `nrr` CLI (paper_2206_03410_b200/cli/nrr_cli.cpp) is driven like
the reference's tools/nrr_cli.cpp: error documents and exit codes 2/3/4 on
the CPU, a full `nrr register` with a JSON report on the GPU.
"""
import json
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2206_03410_b200")


@pytest.fixture(scope="module")
def kats(tmp_path_factory):
    from paper_2206_03410_b200.build import build_library

    build_library()
    exe = str(tmp_path_factory.mktemp("pk") / "pipeline_kats")
    cmd = ["g++", "-O2", "-std=c++20", "-Wall", "-I", os.path.join(ROOT, "include"), "-I",
           os.path.join(ROOT, "tests", "cpp"), "-o", exe, os.path.join(ROOT, "tests/cpp/pipeline_kats.cpp"),
           "-L", LIBDIR, "-lnrr_b200", "-Wl,-rpath," + LIBDIR]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-4000:]
    return exe


@pytest.fixture(scope="module")
def cli():
    from paper_2206_03410_b200.build import build_cli, build_library

    build_library()
    return build_cli()


def _run_kats(exe, prefix):
    r = subprocess.run([exe, prefix], capture_output=True, text=True, timeout=900)
    print(r.stdout)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert "[FAIL]" not in r.stdout and "[PASS]" in r.stdout


def test_pipeline_host_kats(kats):
    _run_kats(kats, "cpu:")


@pytest.mark.gpu
def test_pipeline_gpu_kats(kats):
    _run_kats(kats, "gpu:")


def _strip_obj(path, nx=10, ny=5, bend=0.0):
    with open(path, "w") as f:
        for j in range(ny):
            for i in range(nx):
                x, y = i / (nx - 1), 0.5 * j / (ny - 1)
                f.write("v %.17g %.17g %.17g\n" % (x, y, bend * np.sin(2 * np.pi * x)))
        for j in range(ny - 1):
            for i in range(nx - 1):
                a = j * nx + i + 1
                f.write("f %d %d %d\nf %d %d %d\n" % (a, a + 1, a + nx + 1, a, a + nx + 1, a + nx))


def _error(r):
    return json.loads(r.stderr.strip().splitlines()[-1])["error"]


def test_cli_errors_and_graph_dump(cli, tmp_path):
    """nrr_cli.cpp:246-278: parse errors are config errors (4), unreadable
    files io errors (2); graph-dump works without a GPU (host graph build)."""
    r = subprocess.run([cli, "register", "-s", "a.obj"], capture_output=True, text=True)
    assert r.returncode == 4 and _error(r)["kind"] == "config" and _error(r)["code"] == 4
    r = subprocess.run([cli, "register", "-s", "a.obj", "-t", "b.obj", "-o", "c.obj", "--gt", "bogus"],
                       capture_output=True, text=True)
    assert r.returncode == 4
    r = subprocess.run([cli, "register", "-s", str(tmp_path / "a.obj"), "-t", "b.obj", "-o", "c.obj"],
                       capture_output=True, text=True)
    assert r.returncode == 2 and _error(r)["kind"] == "io"
    r = subprocess.run([cli, "metrics", "--deformed", "x.obj"], capture_output=True, text=True)
    assert r.returncode == 2
    r = subprocess.run([cli, "register", "--help"], capture_output=True, text=True)
    assert r.returncode == 0 and "--radius-mult" in r.stdout
    src = str(tmp_path / "s.obj")
    _strip_obj(src)
    r = subprocess.run([cli, "graph-dump", "--in", src, "--radius-mult", "2.5"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    g = json.loads(r.stdout)
    dump = r.stdout
    assert set(g) == {"edges", "influence", "node_indices", "node_positions", "radius", "reg_weights"}
    assert len(g["influence"]) == 50
    assert abs(np.mean([e["c"] for e in g["reg_weights"]]) - 1.0) < 1e-12
    r = subprocess.run([cli, "metrics", "--deformed", src, "--gt-target", src], capture_output=True, text=True)
    assert r.returncode == 0 and json.loads(r.stdout) == {"metrics": {"rmse": 0.0}}
    cfg = tmp_path / "opts.ini"
    cfg.write_text("# options\nin = %s\nradius_mult = 2.5\n" % src)
    r2 = subprocess.run([cli, "graph-dump", "--config", str(cfg)], capture_output=True, text=True)
    assert r2.returncode == 0 and r2.stdout == dump  # CLI11-style key=value config file


@pytest.mark.gpu
def test_cli_register_end_to_end(cli, tmp_path):
    """`nrr register` (nrr_cli.cpp:149-192 -> run_pipeline) on the B200:
    report schema of proj/README.md:158-178, deterministic apart from timings."""
    src, tgt = str(tmp_path / "s.obj"), str(tmp_path / "t.obj")
    _strip_obj(src, 16, 8)
    _strip_obj(tgt, 16, 8, bend=0.04)
    docs = []
    for tag in ("a", "b"):
        out, rep = str(tmp_path / ("o_%s.obj" % tag)), str(tmp_path / ("r_%s.json" % tag))
        r = subprocess.run([cli, "register", "-s", src, "-t", tgt, "-o", out, "--report", rep, "--gt", "index",
                            "--seed", "3"], capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stderr
        d = json.load(open(rep))
        assert set(d) == {"config", "graph", "normalization", "stages", "solver", "metrics", "timings"}
        assert d["solver"]["total_iterations"] == sum(len(s["iterations"]) for s in d["stages"])
        assert d["metrics"]["rmse"] < 0.05
        for s in d["stages"]:
            e = [it["E"] for it in s["iterations"]]
            assert all(b <= a * (1 + 1e-12) for a, b in zip(e, e[1:]))  # E never increases in a stage
        d.pop("timings")
        d.pop("config")
        docs.append(json.dumps(d, sort_keys=True))
    assert docs[0] == docs[1]
    assert open(str(tmp_path / "o_a.obj")).read() == open(str(tmp_path / "o_b.obj")).read()
