"""Seeded synthetic inputs shared by both sides of the parity contract (content generator, configs, op scripts,
replay dispatch).  Holds none of the method's arithmetic."""
