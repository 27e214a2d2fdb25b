"""Runner layer: time loops (drop-in for pkg/src/micromacro/runner/)."""
