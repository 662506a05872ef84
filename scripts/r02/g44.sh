# round 2, call 44 (1 GPU): g42 (FFMA2(c, lap, +0) fast form A/B + GPU tests) and g43 (e2e vs NUMA placement)
bash scripts/r02/g42.sh
bash scripts/r02/g43.sh
