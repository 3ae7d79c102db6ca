"""phasesync.chaossim -- reference import name kept so that
reference code importing it resolves.  The coupled Rossler-Lorenz simulator is
validation science on N = 2 signals with no N^2 work; this B200 build covers
the PLV-family hot path only, so every operation raises
NotImplementedError naming that scope."""

_SCOPE = ("phasesync.chaossim.{} (SPEC.md:281-377) is outside this build's scope: it implements the "
          "PLV / iPLV / ciPLV hot path (DESIGN.md section 7)")


def _out_of_scope(name):
    def f(*args, **kwargs):
        raise NotImplementedError(_SCOPE.format(name))
    f.__name__ = name
    f.__doc__ = _SCOPE.format(name)
    return f


rossler_derivative = _out_of_scope("rossler_derivative")
lorenz_driven_derivative = _out_of_scope("lorenz_driven_derivative")
integrate_coupled = _out_of_scope("integrate_coupled")
linear_mix = _out_of_scope("linear_mix")
coupling_sweep = _out_of_scope("coupling_sweep")
