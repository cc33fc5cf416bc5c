cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
grep -E "MemTotal|MemAvailable" /proc/meminfo
nvidia-smi --query-gpu=memory.total,memory.used --format=csv
avail_gb=$(awk '/MemAvailable/ {print int($2/1048576)}' /proc/meminfo)
sizes="${SIZES:-20 200}"
if [ "$avail_gb" -gt 300 ]; then sizes="20 200 1000"; fi
echo "sizes: $sizes"
timeout 1500 python tools/bench_csr_build.py $sizes 2>&1 | tee gpurun_out/csr_build.jsonl
