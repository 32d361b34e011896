python - <<'PY'
import paper_2202_11819_b200 as j3d
with j3d.Jacobi3D((512, 512, 512), odf=8, variant="direct", launch="persistent") as ctx:
    ctx.init("hash", seed=1)
    ctx.iterate(100)
    print(ctx.residual(), ctx.checksum())
    u = ctx.gather_local()
    print(u.shape, u.dtype)
PY
