"""Reference-side integrations of the B200 path (the reference is the caller)."""
