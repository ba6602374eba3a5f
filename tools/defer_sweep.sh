for d in 0 0.5 1 2 4; do echo "defer $d"; EXTRA="--defer $d" CONFIGS="cfg2 cfg3 cfg4 cfg5" STEPS=8 bash tools/quick_bench.sh | cut -c1-60; done
