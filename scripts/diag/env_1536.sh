# 1536^3 default workload: TMA L2 hint / promotion / tile order (environment hooks only), alternating with the default
B='--steps 50 --warmup 5'
python scripts/sweep.py "$B" "J3D_TMA_HINT=2 $B" "J3D_L2PROMO=256 $B" "J3D_L2PROMO=64 $B" "$B" "J3D_TILE_ORDER=2 $B" "J3D_TILE_ORDER=3 $B" "J3D_TMA_HINT=1 $B" "$B" "J3D_TMA_HINT=2 $B" "J3D_L2PROMO=256 $B" "$B"
