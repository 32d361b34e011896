# fine384_odf64 batched (96^3 blocks, one launch per iteration): z chunk, tail split, TMA L2 hint, graphs
B='--workload fine384_odf64 --launch batched --steps 200'
python scripts/sweep.py "$B" "J3D_ZCHUNK=12 $B" "J3D_ZCHUNK=24 $B" "J3D_ZCHUNK=32 $B" "J3D_ZCHUNK=48 $B" \
  "J3D_TAILSPLIT=2 $B" "J3D_ZCHUNK=24 J3D_TAILSPLIT=2 $B" "J3D_ZCHUNK=32 J3D_TAILSPLIT=2 $B" \
  "J3D_TMA_HINT=1 $B" "J3D_TMA_HINT=2 $B" "J3D_TILE=19 $B" "J3D_TILE=24 $B" "J3D_TILE=15 $B" \
  "$B --graph 1" "J3D_ZCHUNK=24 $B --graph 1" "J3D_ZCHUNK=32 $B --graph 1" "$B"
