# Beamer switch constant (EngineOptions.alpha) across configs
for a in ${ALPHAS:-4 8 16 32}; do echo "alpha $a"; EXTRA="--alpha $a" CONFIGS="${CONFIGS:-cfg2 cfg3 cfg4 cfg5}" STEPS=8 bash tools/quick_bench.sh; done
