"""Drop-in shim: `import genopt` (and `python -m genopt`) resolve to the
B200-native package paper_2603_19163_b200, so programs, scripts and
subprocess callers written for the reference run unchanged once this
directory is on the path.  See INTEGRATION.md."""
import paper_2603_19163_b200 as _impl

_impl.install_genopt_alias()
