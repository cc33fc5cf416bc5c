cd $GRAFT_REPO_ROOT
for kn in "PDLP_NO_L2_PERSIST=1" "X=1"; do
  for c in C2 C3; do echo "=== $c $kn"; env $kn ENGINE=2 timeout 300 python tools/micro.py $c 2>&1 | grep -v copy; done
done
python - <<'PY'
import torch
p = torch.cuda.get_device_properties(0)
print("L2", p.L2_cache_size, "persisting max", getattr(p, "persisting_l2_cache_max_size", None))
PY
