"""Route the reference package's own hot-path callables through this library.

``install_into_reference(fpmat)`` rebinds the names the reference modules
imported at load time (polmat, appint, kernel,
fraction, solve), so the reference's L4 callers (kernel bases, fraction
reconstruction, solvers) run on the GPU unchanged.  Results are wrapped back
into ``fpmat.polmat.PolMat`` objects.
"""


def _wrap(ref_polmat_cls, fn):
    def inner(*args, **kwargs):
        out = fn(*args, **kwargs)
        return ref_polmat_cls(out.ctx, out.rows, ncols=out.n)

    inner.__name__ = getattr(fn, "__name__", "wrapped")
    inner.__doc__ = getattr(fn, "__doc__", None)
    return inner


def install_into_reference(fpmat_pkg=None):
    """Rebind fpmat's pm_mul / _pm_middle / pmbasis / mbasis / pm_intbasis /
    m_intbasis / eval_polmat_points to the B200 path.

    Returns a dict {module.name: original} that ``uninstall`` restores."""
    import importlib

    from . import appint, polmat

    if fpmat_pkg is None:
        fpmat_pkg = importlib.import_module("fpmat")
    name = fpmat_pkg.__name__
    ref_polmat = importlib.import_module(name + ".polmat")
    RefPolMat = ref_polmat.PolMat
    repl = {
        "pm_mul": _wrap(RefPolMat, polmat.pm_mul),
        "_pm_middle": _wrap(RefPolMat, polmat._pm_middle),
        "pm_middle_product": _wrap(RefPolMat, polmat.pm_middle_product),
        "pmbasis": _wrap(RefPolMat, appint.pmbasis),
        "mbasis": _wrap(RefPolMat, appint.mbasis),
        "pm_intbasis": _wrap(RefPolMat, appint.pm_intbasis),
        "m_intbasis": _wrap(RefPolMat, appint.m_intbasis),
        "eval_polmat_points": appint.eval_polmat_points,
    }
    # import every module first so none binds an already-replaced name
    mods = []
    for mod in ("polmat", "appint", "kernel", "fraction", "solve"):
        try:
            mods.append(importlib.import_module(f"{name}.{mod}"))
        except Exception:
            continue
    saved = {}
    for m in mods:
        for attr, fn in repl.items():
            if hasattr(m, attr):
                saved[(m.__name__, attr)] = getattr(m, attr)
                setattr(m, attr, fn)
    return saved


def uninstall(saved):
    import importlib

    for (modname, attr), fn in saved.items():
        setattr(importlib.import_module(modname), attr, fn)
