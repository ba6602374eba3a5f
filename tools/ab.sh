# same-box A/B: the working tree vs the committed build in _ab/ (git-ignored copy)
# usage: CONFIGS="cfg2 cfg4" ROUNDS=2 bash tools/ab.sh
for r in $(seq ${ROUNDS:-2}); do
  echo "== new"; bash tools/quick_bench.sh
  echo "== old"; (cd _ab && bash tools/quick_bench.sh)
done
