# ring-depth / selection-CTA sweep of the fused step (timeline span + bench value)
cd $GRAFT_REPO_ROOT
for st in 2 3 4 6; do
  echo "== LYC_STAGES=$st"
  LYC_STAGES=$st timeout 300 python scripts/step_timeline.py 2>&1 | grep -E "^  [0-4] |^  7 |span"
done
