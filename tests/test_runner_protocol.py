"""Runner wire protocol (v1) over real stdio, with the GPU-free stub backend, and the
unmodified reference ``ktune runner-check`` / ``ktune tune`` driving it when the reference is
importable (this container; skipped elsewhere)."""
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
SPACES = ROOT / "paper_2505_03780_b200" / "spaces"
REF = Path("/root/reference/pkg/src")
RUNNER = [sys.executable, "-m", "paper_2505_03780_b200.runner"]


def spawn(*extra):
    env = dict(os.environ, PYTHONPATH=str(ROOT))
    return subprocess.Popen([*RUNNER, *extra], stdin=subprocess.PIPE, stdout=subprocess.PIPE,
                            stderr=subprocess.PIPE, text=True, env=env, cwd=ROOT)


def talk(proc, msgs):
    out = []
    for m in msgs:
        proc.stdin.write((m if isinstance(m, str) else json.dumps(m)) + "\n")
        proc.stdin.flush()
        if isinstance(m, dict) and m.get("type") == "shutdown":
            break
        out.append(json.loads(proc.stdout.readline()))
    return out


def test_hello_evaluate_shutdown_stub():
    p = spawn("--binding", str(SPACES / "prefill.binding.json"), "--protocol", "1", "--backend", "stub")
    cfg = dict(BLOCK_M=256, BLOCK_N=128, num_warps=4, num_stages=3, waves_per_eu=1, PRE_LOAD_V=False)
    hello, res, bad, unk, nojs, miss = talk(p, [
        {"type": "hello", "protocol": 1},
        {"type": "evaluate", "config": cfg, "shape": {"op": "prefill", "batch_size": 1, "seq_len": 512}, "warmups": 1,
         "reps": 4},
        {"type": "evaluate", "config": cfg, "reps": 0, "shape": {}},
        {"type": "frobnicate"},
        "not json",
        {"type": "evaluate", "config": {"BLOCK_M": 128}, "shape": {"op": "prefill"}},
        {"type": "shutdown"},
    ])
    assert hello["type"] == "hello" and hello["protocol"] == 1
    fp = hello["fingerprint"]
    assert len(fp) == 8 and all(fp[k] not in ("", None) for k in fp)
    assert "evaluate" in hello["capabilities"]
    assert res["status"] == "ok" and len(res["latencies_ms"]) == 4 and all(v > 0 for v in res["latencies_ms"])
    assert bad["status"] == "error" and unk["status"] == "error" and nojs["status"] == "error"
    assert miss["status"] == "error" and "missing space parameter" in miss["reason"]
    assert p.wait(timeout=10) == 0


def test_protocol_version_refused():
    p = spawn("--binding", str(SPACES / "prefill.binding.json"), "--protocol", "2", "--backend", "stub")
    assert p.wait(timeout=10) == 1


def test_bad_binding_refused(tmp_path):
    b = tmp_path / "b.json"
    b.write_text(json.dumps({"op": "prefill", "space_file": str(SPACES / "flash_attention.space.json"),
                             "config_params": {"BLOCK_M": "BLOCK_M"}}))
    p = spawn("--binding", str(b), "--protocol", "1", "--backend", "stub")
    assert p.wait(timeout=10) == 1
    assert "not mapped" in p.stderr.read()


def test_fingerprint_space_digest_is_ktune_digest():
    from paper_2505_03780_b200 import configspace as CS
    p = spawn("--binding", str(SPACES / "decode.binding.json"), "--protocol", "1", "--backend", "stub")
    (hello,) = talk(p, [{"type": "hello", "protocol": 1}, {"type": "shutdown"}])
    assert hello["fingerprint"]["space_digest"] == CS.parse_space_file(SPACES / "paged_decode.space.json").digest
    p.wait(timeout=10)


needs_ref = pytest.mark.skipif(not (REF / "ktune").is_dir(), reason="reference ktune not present")


def ktune(*args, cwd=None):
    env = dict(os.environ, PYTHONPATH=f"{REF}:{ROOT}")
    return subprocess.run([sys.executable, "-m", "ktune", *args], capture_output=True, text=True, env=env,
                          cwd=cwd or ROOT, timeout=300)


@needs_ref
def test_unmodified_ktune_runner_check_passes():
    cmd = f"{sys.executable} -m paper_2505_03780_b200.runner --binding {SPACES / 'prefill.binding.json'} " \
          f"--protocol 1 --backend stub"
    r = ktune("runner-check", "--runner", cmd, "--space", str(SPACES / "flash_attention.space.json"),
              "--shape", "op=prefill,batch_size=1,seq_len=512,num_q_heads=32,num_kv_heads=8,head_dim=128")
    assert r.returncode == 0, r.stdout + r.stderr
    assert "assertions passed" in r.stdout and "[FAIL]" not in r.stdout


@needs_ref
def test_unmodified_ktune_tune_drives_runner_and_caches(tmp_path):
    cmd = f"{sys.executable} -m paper_2505_03780_b200.runner --binding {SPACES / 'decode.binding.json'} " \
          f"--protocol 1 --backend stub"
    args = ["tune", "--space", str(SPACES / "paged_decode.space.json"), "--runner", cmd, "--shape",
            "op=decode,batch_size=64,seq_len=4096,num_q_heads=32,num_kv_heads=8,head_dim=128,block_size=16",
            "--cache-dir", str(tmp_path / "cache"), "--json"]
    r1 = ktune(*args)
    assert r1.returncode == 0, r1.stdout + r1.stderr
    r2 = ktune(*args)
    assert r2.returncode == 0, r2.stdout + r2.stderr
    doc = json.loads(r2.stdout)
    assert json.dumps(doc).count("cache") >= 1
