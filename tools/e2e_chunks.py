import os, sys, subprocess
for c in ["262144", "524288", "1048576", "2097152", "4194304"]:
    env = dict(os.environ, KT_HOST_CHUNK=c)
    out = subprocess.run([sys.executable, "tools/e2e_sweep.py"], env=env, capture_output=True, text=True).stdout
    line = [l for l in out.splitlines() if "work= 128" in l]
    print("chunk", c, line[0] if line else out[-300:])
