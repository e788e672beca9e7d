"""Run tests/slab_worker.py on `world` local processes (gloo, 127.0.0.1) and collect their JSON lines."""
import json
import os
import socket
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def run(world, *args, timeout=600, one_gpu_per_rank=False):
    port = free_port()
    procs = []
    for r in range(world):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE=str(world), MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port),
                   LOCAL_RANK=str(r) if one_gpu_per_rank else "0")
        procs.append(subprocess.Popen([sys.executable, os.path.join(HERE, "slab_worker.py"), *map(str, args)],
                                      env=env, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True))
    results = {}
    errs = []
    for p in procs:
        try:
            o, e = p.communicate(timeout=timeout)
        except subprocess.TimeoutExpired:
            for q in procs:
                q.kill()
            raise
        errs.append(e[-3000:])
        for line in o.splitlines():
            if line.startswith("RESULT "):
                d = json.loads(line[7:])
                results[d["rank"]] = d
    if len(results) != world:
        raise RuntimeError("slab worker failed:\n" + "\n----\n".join(errs))
    return [results[r] for r in range(world)]
