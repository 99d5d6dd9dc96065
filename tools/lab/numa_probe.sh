nvidia-smi topo -m 2>&1 | head -8
lscpu | grep -i "numa\|socket\|model name" | head -8
python - <<'PY'
import pynvml as n
n.nvmlInit(); h=n.nvmlDeviceGetHandleByIndex(0)
aff=n.nvmlDeviceGetCpuAffinity(h, 4)
cpus=[]
for w,word in enumerate(aff):
    for b in range(64):
        if word>>b & 1: cpus.append(w*64+b)
print("gpu0 local cpus:", cpus[:4], "...", len(cpus))
try:
    print("numa node mem affinity:", n.nvmlDeviceGetMemoryAffinity(h, 4, 0))
except Exception as e: print("mem aff n/a", e)
PY
echo "== default"; ./tools/lab/d2h_bw
CPUS=$(python -c "
import pynvml as n
n.nvmlInit(); h=n.nvmlDeviceGetHandleByIndex(0)
aff=n.nvmlDeviceGetCpuAffinity(h, 4)
print(','.join(str(w*64+b) for w,word in enumerate(aff) for b in range(64) if word>>b&1))")
echo "== taskset local $CPUS"; taskset -c $CPUS ./tools/lab/d2h_bw
echo "== other cpus"; nproc; taskset -c 0 ./tools/lab/d2h_bw
