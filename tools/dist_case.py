"""Run one slab-decomposed case against the single-GPU step (debug helper):
    python tools/dist_case.py WORLD '{"spec": {...}, "seed": 0, "steps": 3}'
Prints the first step/array that differs."""
import json
import os
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import test_dist_gpu as T  # noqa: E402

world, case = int(sys.argv[1]), json.loads(sys.argv[2])
out = os.path.join(tempfile.mkdtemp(), "d.json")
cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
       "--master-addr=127.0.0.1", f"--master-port={T._free_port()}",
       os.path.join(ROOT, "tests", "_dist_gpu_worker.py"), out, json.dumps(case)]
r = subprocess.run(cmd, capture_output=True, text=True, env=dict(os.environ, MASTER_ADDR="127.0.0.1"))
if r.returncode:
    print(r.stdout[-3000:], r.stderr[-3000:])
    sys.exit(1)
got = json.load(open(out))["steps"]
exp = T._single(case)
for s, (g, e) in enumerate(zip(got, exp)):
    bad = [k for k in e if g[k] != e[k]]
    print(f"world {world} {case['spec']} step {s + 1}: {'OK' if not bad else bad} "
          f"its {g['its']}/{e['its']} res {g['res']}/{e['res']}")
